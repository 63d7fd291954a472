"""Rounding-noise study of B2 at config 4 (diagnostic): exact ||A - A_hat||_F of
the GPU compression under 1-ulp perturbations of the grid coordinates, and
the exact distances between the perturbed results (ublr_frob_error /
ublr_frob_diff). python tools/b2_noise.py [c4|c3]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2501_05528_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
mid = {"c4": "B2", "c3": "A1"}[cfg]
pts = P.grid_points(256, 2)
tess = P.build_tessellation(pts, 256)
diag = -np.log(0.5 / 256)
op0 = P.KernelOperator(pts, "log", diag)
variants = {"base": pts.coords, "+1ulp": np.nextafter(pts.coords, 2.0), "-1ulp": np.nextafter(pts.coords, -1.0),
            "+1ulp x": np.stack([np.nextafter(pts.coords[:, 0], 2.0), pts.coords[:, 1]], 1),
            "+2ulp": np.nextafter(np.nextafter(pts.coords, 2.0), 2.0)}
reps = {}
A_fro = None
for name, c in variants.items():
    rep, _ = P.compress(P.KernelOperator(c, "log", diag), tess, 40, mid, p=10, stream=P.RandomStream(7),
                        compute_error=False)
    fr = P.frobenius_error(op0, rep)      # error against the UNPERTURBED A
    A_fro = fr.ref_fro
    reps[name] = rep
    print(f"{cfg} {mid} {name:8s} ||A - A_hat||_F / ||A||_F = {fr.fro / A_fro:.4e}", flush=True)
base = reps["base"]
for name, rep in reps.items():
    if name != "base":
        print(f"   ||A_hat(base) - A_hat({name})||_F / ||A||_F = {P.frobenius_distance(base, rep).fro / A_fro:.3e}")
