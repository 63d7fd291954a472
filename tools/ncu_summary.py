"""Key counters + top stall reasons from an ncu report (run here, no GPU)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for k in keys:
    if k in d:
        print(f"{k:80s} {d[k]} {units[hdr.index(k)]}")
st = [(h, v) for h, v in d.items() if h.startswith("smsp__average_warp_latency_issue_stalled_") or
      (h.startswith("smsp__warp_issue_stalled_") and h.endswith("_per_warp_active.pct"))]
st = sorted(((h, float(v)) for h, v in st if v.replace('.', '', 1).isdigit()), key=lambda x: -x[1])[:10]
print("top stalls:")
for h, v in st:
    print(f"  {h:78s} {v:.2f}")
