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
def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


# stall reasons: average warps stalled per issued instruction (the ratio ncu's
# "Warp State Statistics" section plots), largest first
pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
st = [(h[len(pre):-len(suf)], num(v)) for h, v in d.items() if h.startswith(pre) and h.endswith(suf)]
st = sorted((x for x in st if x[1] is not None), key=lambda x: -x[1])[:10]
print("top stalls (warps stalled per issued instruction):")
for h, v in st:
    print(f"  {h:40s} {v:.3f}")
samp = [(h[len("smsp__pcsamp_warps_issue_stalled_"):], num(v)) for h, v in d.items()
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
samp = [x for x in samp if x[1] is not None]
tot = sum(v for _, v in samp)
if tot > 0:
    print("pc-sampling stall share:")
    for h, v in sorted(samp, key=lambda x: -x[1])[:8]:
        print(f"  {h:40s} {100 * v / tot:.1f} %")
