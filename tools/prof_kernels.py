"""Small single-launch cases for ncu captures of the hot kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2501_05528_b200 as P
from paper_2501_05528_b200.bases import draw_test_blocks, tagged_sketch
from paper_2501_05528_b200.tessellation import device_tess

which = sys.argv[1:] or ["sketch", "apply", "coupling"]
torch.cuda.set_device(0)
pts = P.grid_points(256, 2)
tess = P.build_tessellation(pts, 256)
dt = device_tess(tess, torch.device("cuda"))
op = P.KernelOperator(pts, "inv", 512.0)
if "sketch" in which:
    plan = P.plan_tagging(tess, 0, "gaussian", P.RandomStream(7).child(1))
    G = draw_test_blocks(dt, P.RandomStream(1), 0, 64)
    H = draw_test_blocks(dt, P.RandomStream(1), 1, 64)
    T = torch.from_numpy(plan.matrix.entries).cuda()
    for _ in range(2):
        tagged_sketch(op, dt, T, plan.matrix.entries, G, H, 64)
if "apply" in which:
    X = torch.randn(dt.n, 1024, dtype=torch.float64, device="cuda")
    for _ in range(2):
        op.apply_device(X, dt.perm)
if "coupling" in which:
    from paper_2501_05528_b200.bases import BlockBases
    from paper_2501_05528_b200.reconstruction import direct_core
    U = torch.randn(dt.n, 48, dtype=torch.float64, device="cuda")
    bs = BlockBases(dt, U, U.clone(), 48, "tag", (0, 0))
    for _ in range(2):
        direct_core(op, tess, bs)
torch.cuda.synchronize()
print("ok")
