"""Full-size golden fixtures for configs 3 and 4 from the UNMODIFIED reference.

The reference compressor runs here with a chunked, multithreaded on-the-fly
operator for the -log|x-y| kernel (the 34 GB matrix is never formed; the
adapter only provides shape/apply/apply_adjoint). Outputs are
stored as probes of the assembled operator (A_hat W, A_hat^T W for a fixed
Gaussian W) so the files stay small. Takes tens of minutes per config:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_large.py c3 [c4]
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from ublr import RandomStream, build_tessellation, compress, grid_points  # noqa: E402

from oracle.operators import KernelOp  # noqa: E402  (shape/apply adapter only)

OUT = os.path.dirname(os.path.abspath(__file__))


def probe_vec(n, salt):
    return np.random.default_rng(1000 + salt).standard_normal(n)


def frob_kernel(op):
    n = op.shape[0]
    tot = 0.0
    for lo in range(0, n, 2048):
        blk = op._rows_block(lo, min(lo + 2048, n)) if hasattr(op, "_rows_block") else None
        if blk is None:
            from oracle.operators import kernel_block
            blk = kernel_block(op.coords, np.arange(lo, min(lo + 2048, n)), np.arange(n), op.kind, op.diag)
        tot += float(np.sum(blk * blk))
    return np.sqrt(tot)


def run(name):
    per, b = 256, 256
    pts = grid_points(per, 2)
    tess = build_tessellation(pts, b)
    op = KernelOp(pts.coords, "log", -np.log(0.5 / per), chunk=256)
    k, p, mid = 40, 10, {"c3": "A1", "c4": "B2"}[name]
    t0 = time.time()
    rep, report = compress(op, tess, k, method_id=mid, p=p, stream=RandomStream(7), compute_error=False)
    t1 = time.time()
    W = np.stack([probe_vec(tess.n_points, 10 + c) for c in range(3)], axis=1)
    out = {
        "N": tess.n_points, "b": b, "k": k,
        "Ahat_W": rep.apply(W), "Ahat_tW": rep.apply_adjoint(W),
        "A_W": op.apply(W),
        "A_fro": frob_kernel(op),
        "matvecs": np.array([[report.matvecs.get(ph, {"A": 0})["A"], report.matvecs.get(ph, {"Astar": 0})["Astar"]]
                             for ph in ("I", "II", "III")]),
        "storage_entries": report.storage_entries,
        "ref_seconds": np.array([t1 - t0] + [report.times_s.get(ph, np.nan) for ph in ("I", "II", "III")]),
        "ranks": rep.effective_ranks,
    }
    np.savez_compressed(os.path.join(OUT, f"{name}_{mid}.npz"), **out)
    print(name, mid, "reference seconds", t1 - t0, report.times_s, flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c3"]:
        run(name)
