"""Diagnostic (not product): rounding sensitivity of B2 at config-4 size.
Runs the GPU B2 compression twice — exact grid coordinates and coordinates
perturbed by one ulp (A entries move by ~1e-16 relative) — and reports the
change of A_hat, next to the difference from the reference fixture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2501_05528_b200 as P
from cases import GOLDEN, probe_vec

name, mid = (sys.argv[1], sys.argv[2]) if len(sys.argv) > 2 else ("c4_B2", "B2")
g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
pts = P.grid_points(256, 2)
tess = P.build_tessellation(pts, 256)
W = np.stack([probe_vec(tess.n_points, 10 + c) for c in range(3)], axis=1)
scale = float(g["A_fro"]) * np.sqrt(3)
outs = []
for label, coords in (("exact", pts.coords), ("1-ulp", np.nextafter(pts.coords, 2.0))):
    op = P.KernelOperator(coords, "log", -np.log(0.5 / 256))
    rep, _ = P.compress(op, tess, 40, mid, p=10, stream=P.RandomStream(7), compute_error=False)
    AW = rep.apply(W)
    outs.append(AW)
    print(label, "dAhat vs reference", np.linalg.norm(AW - g["Ahat_W"]) / scale,
          "approx err", np.linalg.norm(g["A_W"] - AW) / scale)
print("rounding sensitivity |A_hat(exact) - A_hat(1-ulp coords)| / |A|:", np.linalg.norm(outs[0] - outs[1]) / scale)
print("reference approx err", np.linalg.norm(g["A_W"] - g["Ahat_W"]) / scale)
