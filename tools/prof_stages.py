"""Per-entry-point / per-GEMM-shape GPU time of one compression (CUDA events).
Diagnostic only: python tools/prof_stages.py c3"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import _lib, workloads as W

wl = W.build(sys.argv[1] if len(sys.argv) > 1 else "c3")
run = lambda: P.compress(wl.op, wl.tess, wl.k, wl.method, p=wl.p, stream=P.RandomStream(7), compute_error=False)
run(); torch.cuda.synchronize()
orig = _lib.call
shapes = {}
def call(name, *args, **kw):
    if name == "ublr_gemm_batched":
        key = f"gemm t{args[0]}{args[1]} M{args[2]} N{args[3]} K{args[4]} b{args[22]}"
    else:
        key = name
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); orig(name, *args, **kw); b.record()
    shapes.setdefault(key, []).append((a, b, _lib._work_of(name, args)))
_lib.call = call
import paper_2501_05528_b200.dense as D
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); run(); t1.record(); torch.cuda.synchronize()
tot = t0.elapsed_time(t1)
rows = []
for k, v in shapes.items():
    ms = sum(a.elapsed_time(b) for a, b, _ in v)
    fl = sum(w for _, _, w in v)
    rows.append((ms, len(v), k, fl / ms / 1e9 if ms else 0))
rows.sort(reverse=True)
print(f"total {tot:.1f} ms; kernels {sum(r[0] for r in rows):.1f} ms")
agg = {}
for ms, n, k, tf in rows:
    agg.setdefault(k.split(" ")[0], [0, 0])
    agg[k.split(" ")[0]][0] += ms; agg[k.split(" ")[0]][1] += n
for k, (ms, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:30s} {n:6d} {ms:9.2f} ms")
print("--- top shapes")
for ms, n, k, tf in rows[:45]:
    print(f"{ms:9.2f} ms {n:5d}x  {tf:6.2f} TF/s  {k}")
