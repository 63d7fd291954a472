"""Golden fixtures for the tagging options (null-vector optimisation,
extra_samples, equidistributed / haar rows, extra tagging columns), made by
running the UNMODIFIED reference package in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_options.py

Writes tests/golden/plans_options.npz (tagging plans) and
tests/golden/opt_<case>.npz (compressions of the 32 x 32 log-kernel grid).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import OUT, log_matrix, save_rep  # noqa: E402
from ublr import DenseOperator, RandomStream, build_tessellation, compress, grid_points, plan_tagging  # noqa: E402
from ublr.linalg import null_basis  # noqa: E402

# name -> (per_axis, b, extra_cols, distribution, optimize)
PLANS = {
    "g16_opt": (32, 16, 0, "gaussian", True),
    "g64_opt": (64, 64, 0, "gaussian", True),
    "g16_x2_opt": (32, 16, 2, "gaussian", True),
    "g16_equi": (32, 16, 0, "equidistributed", False),
    "g16_haar_x1": (32, 16, 1, "haar", False),
}

# name -> (method_id, k, p, kwargs)
COMPRESSIONS = {
    "A2_opt": ("A2", 10, 5, {"optimize": True}),
    "A2_xs": ("A2", 10, 5, {"extra_samples": True}),
    "A2_equi": ("A2", 10, 5, {"distribution": "equidistributed"}),
    "A2_haar_x1": ("A2", 10, 5, {"distribution": "haar", "extra_cols": 1}),
    "A2_x2_opt": ("A2", 10, 5, {"extra_cols": 2, "optimize": True}),
    "B2_opt": ("B2", 8, 4, {"optimize": True}),
}


def main():
    plans = {}
    for name, (per, b, xc, dist, opt) in PLANS.items():
        tess = build_tessellation(grid_points(per, 2), b)
        plan = plan_tagging(tess, xc, dist, RandomStream(7).child(1), optimize=opt)
        T = plan.matrix.entries
        plans[f"{name}_T"] = T
        plans[f"{name}_Z"] = np.stack([nv.vector for nv in plan.null_vectors])
        plans[f"{name}_rho"] = plan.rho_base
        if plan.rho_optimized is not None:
            plans[f"{name}_rho_opt"] = plan.rho_optimized
        plans[f"{name}_attempts"] = np.array(plan.attempts)
        # extra_samples combination vector: first column of null_basis (ref/bases.py:177-182)
        X = np.stack([null_basis(T[nb, :], T.shape[1] - len(nb))[:, 0] if T.shape[1] - len(nb) >= 2
                      else plan.null_vectors[i].vector for i, nb in enumerate(tess.neighbor_lists)])
        plans[f"{name}_X"] = X
        print(name, plan.attempts, None if plan.rho_optimized is None else np.nanmax(plan.rho_optimized))
    np.savez_compressed(os.path.join(OUT, "plans_options.npz"), **plans)

    pts = grid_points(32, 2)
    tess = build_tessellation(pts, 16)
    A = log_matrix(pts, 1.0 / 32)
    for name, (mid, k, p, kw) in COMPRESSIONS.items():
        rep, report = compress(DenseOperator(A), tess, k, method_id=mid, p=p, stream=RandomStream(7), **kw)
        extra = {}
        if report.aspect_ratios and "optimized" in report.aspect_ratios:
            extra["rho_opt_max"] = np.array(report.aspect_ratios["optimized"]["max"])
        save_rep(f"opt_{name}", rep, report, A, extra)


if __name__ == "__main__":
    main()
