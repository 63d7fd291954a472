"""Small end-to-end cases for compute-sanitizer runs (memcheck / racecheck /
synccheck), one process per case:

    compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_case.py c2

c1, c2: the BASELINE configs (dense synthetic d=1; -log kernel 64 x 64 grid).
c5s:    the config-5 code path at a sanitizer-friendly size — 1/r kernel,
        m = 256, k = 48, p = 16, A2, block rows sharded 8 ways with the
        shifted (negative-offset) shard pointers, one rank's share
        (shard 3) after the other shards' V rows.
c3s:    the config-3 A1 path (block-nullification null space, -log kernel,
        m = 256) on a 128 x 128 grid (64 boxes).
b2s:    type B (B2) on a ragged 50 x 50 grid.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import workloads as W

case = sys.argv[1] if len(sys.argv) > 1 else "c2"
if case in ("c1", "c2"):
    wl = W.build(case)
    P.compress(wl.op, wl.tess, wl.k, wl.method, p=wl.p, stream=P.RandomStream(7), compute_error=True)
elif case == "c5s":
    from paper_2501_05528_b200.distributed import phase1_local, phase23_local, shard_ranges
    per = 256
    pts = P.grid_points(per, 2)
    tess = P.build_tessellation(pts, 256)
    op = P.KernelOperator(pts, "inv", 2.0 * per)
    shards = shard_ranges(tess, 8, 48)
    st = P.RandomStream(7)
    plan = P.plan_tagging(tess, 0, "gaussian", st.child(1), device=True)
    Vs = [phase1_local(op, tess, 48, 16, st, sh, plan)[2] for sh in shards]
    _, U, V, dt = phase1_local(op, tess, 48, 16, st, shards[3], plan)
    phase23_local(op, 48, shards[3], dt, U, torch.cat(Vs, 0))
    host = torch.empty((shards[3].K1 - shards[3].K0, int(dt.roff(48)[0][-1])), dtype=torch.float64,
                       pin_memory=True)
    phase23_local(op, 48, shards[3], dt, U, torch.cat(Vs, 0), core_out=host, panel_blocks=5)
elif case == "c3s":
    per = 128
    pts = P.grid_points(per, 2)
    tess = P.build_tessellation(pts, 64)
    P.compress(P.KernelOperator(pts, "log", -np.log(0.5 / per)), tess, 40, "A1", p=10, stream=P.RandomStream(7),
               compute_error=False)
elif case == "b2s":
    per = 50
    pts = P.grid_points(per, 2)
    tess = P.build_tessellation(pts, 16)
    P.compress(P.KernelOperator(pts, "log", -np.log(0.5 / per)), tess, 20, "B2", p=10, stream=P.RandomStream(7),
               compute_error=False)
else:
    raise SystemExit(f"unknown case {case}")
torch.cuda.synchronize()
print("ok", case)
