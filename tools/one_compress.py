"""Run `reps` compressions of a BASELINE config (diagnostic / ncu target):
python tools/one_compress.py c3 [reps]   (c5: one rank's share of an 8-way job)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
wl = W.build(cfg)
if cfg == "c5":
    from paper_2501_05528_b200.distributed import phase1_local, phase23_local, shard_ranges
    shards = shard_ranges(wl.tess, 8, wl.k)
    sh = shards[3]
    for _ in range(reps):
        plan, U, V, dt = phase1_local(wl.op, wl.tess, wl.k, wl.p, P.RandomStream(W.COMPRESS_SEED), sh)
        V_all = torch.zeros((dt.n, wl.k), dtype=torch.float64, device="cuda")
        V_all[sh.r0:sh.r1] = V
        phase23_local(wl.op, wl.k, sh, dt, U, V_all)
else:
    for _ in range(reps):
        P.compress(wl.op, wl.tess, wl.k, wl.method, p=wl.p, stream=P.RandomStream(W.COMPRESS_SEED),
                   compute_error=False)
torch.cuda.synchronize()
print("ok", cfg, reps)
