"""Turn gpurun_out/prof (tools/profile_round.sh) into the committed summaries:
profiles/r01/launches_<cfg>.csv + _summary.txt, <capture>_details.txt
(ncu --page details), <capture>_summary.txt (key counters + stalls), and
profiles/traffic_<cfg>.json (DRAM bytes per launch of the bench's dominant
kernel, read by bench.py's roofline)."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# python tools/summarize_profiles.py [dst] : dst defaults to profiles/r02 when
# run here; on the GPU box pass a directory under gpurun_out/ (the .ncu-rep
# files of several full captures exceed what gpurun copies back, so they are
# summarised there and only the text travels)
SRC = os.path.join(ROOT, "gpurun_out", "prof")
DST = os.path.abspath(sys.argv[1]) if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02")
TRAFFIC_DIR = DST if len(sys.argv) > 1 else os.path.join(ROOT, "profiles")
ROUND = os.environ.get("UBLR_PROF_ROUND", "r02")
os.makedirs(DST, exist_ok=True)


def run(args):
    return subprocess.run(args, capture_output=True, text=True).stdout


for cfg in ("c2_bench", "c2", "c3", "c4", "c5"):
    f = os.path.join(SRC, f"launches_{cfg}.csv")
    if os.path.exists(f):
        shutil.copy(f, os.path.join(DST, f"launches_{cfg}.csv"))
        out = run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), f])
        open(os.path.join(DST, f"launches_{cfg}_summary.txt"), "w").write(out)
        print(f"== {cfg}\n" + "\n".join(out.splitlines()[:8]))

# capture -> (bench config, C-ABI entry the bench attributes it to)
CAPS = {"c2_sketch4": ("c2", "ublr_sketch_tagged_pair"), "c2_cnf": (None, "ublr_coupling_nearfield"),
        "c3_apply3": ("c3", "ublr_apply"), "c3_apply4": ("c3", "ublr_apply"), "c3_gemm3": (None, "ublr_gemm_batched"),
        "c3_gen_strip": (None, "ublr_apply_staged"), "c3_apply_gemm3": (None, "ublr_apply_staged"),
        "c4_apply3": ("c4", "ublr_apply"), "c4_apply4": ("c4", "ublr_apply"),
        "c4_sketch4": (None, "ublr_sketch_tagged_comp"), "c5_sketch4": ("c5", "ublr_sketch_tagged_pair"), "c5_coupling3": (None, "ublr_coupling")}
for cap, (cfg, entry) in CAPS.items():
    rep = os.path.join(SRC, f"{cap}.ncu-rep")
    if not os.path.exists(rep):
        continue
    open(os.path.join(DST, f"{cap}_details.txt"), "w").write(run(["ncu", "-i", rep, "--page", "details"]))
    summ = run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep])
    open(os.path.join(DST, f"{cap}_summary.txt"), "w").write(summ)
    raw = run(["ncu", "-i", rep, "--page", "raw", "--csv"])
    rows = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rows[0], rows[2]))
    units = dict(zip(rows[0], rows[1]))

    def nbytes(key):
        v = float(d[key].replace(",", ""))
        u = units.get(key, "byte").lower()
        return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}.get(u, 1)

    rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
    print(f"{cap}: {d.get('Kernel Name', '')[:60]} dram read {rd:.3e} write {wr:.3e}")
    if cfg:
        json.dump({"entry": entry, "kernel": d.get("Kernel Name", "")[:120], "config": cfg,
                   "source": f"profiles/{ROUND}/{cap}_details.txt (ncu --set full --clock-control none, "
                             f"tools/profile_round.sh)",
                   "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr},
                  open(os.path.join(TRAFFIC_DIR, f"traffic_{cfg}.json"), "w"), indent=1)
