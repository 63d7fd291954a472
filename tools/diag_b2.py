"""Diagnostic (not product): sensitivity of the config-4 B2 core solve.
Compares the CholeskyQR2 right-pseudo-inverse core with torch/cuSOLVER SVD and
QR solutions of the same system, and reports the conditioning of V^T Omega."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import typeb
from cases import GOLDEN, probe_vec

stash = {}
orig = typeb.lstsq_right
def spy(LHS, M):
    stash["LHS"], stash["M"] = LHS.clone(), M.clone()
    return orig(LHS, M)
typeb.lstsq_right = spy
pts = P.grid_points(256, 2)
tess = P.build_tessellation(pts, 256)
op = P.KernelOperator(pts, "log", -np.log(0.5 / 256))
rep, _ = P.compress(op, tess, 40, "B2", p=10, stream=P.RandomStream(7), compute_error=False)
g = dict(np.load(os.path.join(GOLDEN, "c4_B2.npz")))
W = np.stack([probe_vec(tess.n_points, 10 + c) for c in range(3)], axis=1)
scale = float(g["A_fro"]) * np.sqrt(3)
def dev(rep_):
    return np.linalg.norm(rep_.apply(W) - g["Ahat_W"]) / scale
print("qr2 core: dAhat vs reference", dev(rep))
print("approx err gpu", np.linalg.norm(g["A_W"] - rep.apply(W)) / scale, "ref", np.linalg.norm(g["A_W"] - g["Ahat_W"]) / scale)
M, LHS = stash["M"], stash["LHS"]
s = torch.linalg.svdvals(M)
print("V^T Omega: shape", tuple(M.shape), "smax", float(s[0]), "smin", float(s[-1]), "cond", float(s[0] / s[-1]))
# SVD pseudo-inverse like the reference (truncate s <= 1e-12 s_max)
U_, S_, Vh = torch.linalg.svd(M, full_matrices=False)
keep = S_ > 1e-12 * S_[0]
Mp = (Vh[keep].T / S_[keep]) @ U_[:, keep].T
core_svd = LHS @ Mp
core0 = rep.core_d.clone()
rep.core_d = core_svd
rep._host = {}
print("svd core: dAhat vs reference", dev(rep), " |core_svd - core_qr2|/|core|",
      float(torch.linalg.norm(core_svd - core0) / torch.linalg.norm(core0)))
