"""Full-size golden fixtures for configs 3 and 4 from the UNMODIFIED reference.

The reference compressor runs here with a chunked, multithreaded on-the-fly
operator for the -log|x-y| kernel (the 34 GB matrix is never formed; the
adapter only provides shape/apply/apply_adjoint). Stored:

* probes of the assembled reference operator, A_hat_ref W and A_hat_ref^T W
  for a fixed Gaussian W with 8 columns (the parity gate
  ||A_hat_gpu - A_hat_ref||_F is estimated from them on the GPU box, where the
  reference's 2 GB output cannot travel);
* EXACT blockwise Frobenius norms computed here, block row by block row:
  ||A||_F, ||A - A_hat_ref||_F and the per-pair ||(A - A_hat_ref)_ij||_F;
* for c4 (B2) also the reference's OWN rounding sensitivity: the unmodified
  reference is run a second time with every grid coordinate moved up by one
  ulp (np.nextafter(coords, 2), A entries change by ~1e-16 relative) and the
  exact ||A_hat_ref - A_hat_ref'||_F (total and per pair) is stored, with the
  perturbed run's own exact error ||A - A_hat_ref'||_F, and the exact
  errors over a family of five 1-ulp coordinate perturbations (base, +1, -1,
  +1 on axis 0, +2 ulp). The GPU gates for B2 are anchored on these numbers,
  not on the GPU's own.

Takes ~40 min for c3 and ~35 min for c4 (two reference runs) on 8 cores:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_large.py c4 c3
"""

from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from ublr import RandomStream, build_tessellation, compress, grid_points  # noqa: E402

from oracle.operators import KernelOp, kernel_block  # noqa: E402  (shape/apply adapter only)

OUT = os.path.dirname(os.path.abspath(__file__))
N_PROBES = 8


def probe_vec(n, salt):
    return np.random.default_rng(1000 + salt).standard_normal(n)


class BlockRows:
    """Dense block rows of a reference UniformBLR, columns in block order
    (block j occupies columns j*m .. (j+1)*m of the returned m x N array)."""

    def __init__(self, rep):
        self.rep = rep
        tess = rep.tess
        self.b = tess.b
        self.m = int(tess.block_sizes[0])
        self.k = int(rep.effective_ranks[0])
        assert (tess.block_sizes == self.m).all() and (rep.effective_ranks == self.k).all()
        self.V = np.stack(rep.v_blocks)          # (b, m, k)

    def row(self, i):
        b, m, k = self.b, self.m, self.k
        Ci = self.rep.core[i * k:(i + 1) * k].reshape(k, b, k)       # C_ij, j = axis 1
        W = np.einsum("ajc,jmc->ajm", Ci, self.V, optimize=True)     # C_ij V_j^T
        out = self.rep.u_blocks[i] @ W.reshape(k, b * m)
        for j in self.rep.tess.neighbor_lists[i]:
            out[:, j * m:(j + 1) * m] += self.rep.b_blocks[(i, j)]
        return out


def blockwise_norms(tess, coords, diag, reps):
    """Per block pair: ||A_ij||_F^2, ||(A - reps[0])_ij||_F^2 and, with two
    representations, ||(reps[0] - reps[1])_ij||_F^2 and ||(A - reps[1])_ij||_F^2
    (exact, in fp64)."""
    b = tess.b
    cols = np.concatenate(tess.blocks)
    m = int(tess.block_sizes[0])
    rows_of = [BlockRows(r) for r in reps]
    a2 = np.zeros((b, b))
    e2 = np.zeros((b, b))
    d2 = np.zeros((b, b))
    f2 = np.zeros((b, b))

    def one(i):
        A = kernel_block(coords, tess.blocks[i], cols, "log", diag)
        H0 = rows_of[0].row(i)
        a2[i] = np.einsum("rjc,rjc->j", A.reshape(m, b, m), A.reshape(m, b, m))
        D = (A - H0).reshape(m, b, m)
        e2[i] = np.einsum("rjc,rjc->j", D, D)
        if len(rows_of) > 1:
            H1 = rows_of[1].row(i)
            D = (H0 - H1).reshape(m, b, m)
            d2[i] = np.einsum("rjc,rjc->j", D, D)
            D = (A - H1).reshape(m, b, m)
            f2[i] = np.einsum("rjc,rjc->j", D, D)

    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        list(ex.map(one, range(b)))
    return a2, e2, d2, f2


def run(name):
    per, b = 256, 256
    pts = grid_points(per, 2)
    tess = build_tessellation(pts, b)
    diag = -np.log(0.5 / per)
    op = KernelOp(pts.coords, "log", diag, chunk=256)
    k, p, mid = 40, 10, {"c3": "A1", "c4": "B2"}[name]
    t0 = time.time()
    rep, report = compress(op, tess, k, method_id=mid, p=p, stream=RandomStream(7), compute_error=False)
    t1 = time.time()
    print(name, mid, "reference seconds", t1 - t0, report.times_s, flush=True)
    W = np.stack([probe_vec(tess.n_points, 10 + c) for c in range(N_PROBES)], axis=1)
    out = {
        "N": tess.n_points, "b": b, "k": k,
        "Ahat_W": rep.apply(W), "Ahat_tW": rep.apply_adjoint(W),
        "matvecs": np.array([[report.matvecs.get(ph, {"A": 0})["A"], report.matvecs.get(ph, {"Astar": 0})["Astar"]]
                             for ph in ("I", "II", "III")]),
        "storage_entries": report.storage_entries,
        "ref_seconds": np.array([t1 - t0] + [report.times_s.get(ph, np.nan) for ph in ("I", "II", "III")]),
        "ranks": rep.effective_ranks,
    }
    reps = [rep]
    family = {}
    if name == "c4":
        # the reference's own 1-ulp rounding sensitivity (same tessellation,
        # same streams; only the operator's coordinates move), and its exact
        # error over a family of 1-ulp coordinate perturbations (the B2 error
        # at c4 is rounding-noise dominated)
        c = pts.coords
        variants = {"+1ulp": np.nextafter(c, 2.0), "-1ulp": np.nextafter(c, -1.0),
                    "+1ulp x": np.stack([np.nextafter(c[:, 0], 2.0), c[:, 1]], 1),
                    "+2ulp": np.nextafter(np.nextafter(c, 2.0), 2.0)}
        for vname, vc in variants.items():
            t2 = time.time()
            repv, _ = compress(KernelOp(vc, "log", diag, chunk=256), tess, k, method_id=mid, p=p,
                               stream=RandomStream(7), compute_error=False)
            print(name, vname, "perturbed reference seconds", time.time() - t2, flush=True)
            if vname == "+1ulp":
                reps.append(repv)
            else:
                family[vname] = np.sqrt(blockwise_norms(tess, c, diag, [repv])[1].sum())
            del repv
    t3 = time.time()
    a2, e2, d2, f2 = blockwise_norms(tess, pts.coords, diag, reps)
    print(name, "blockwise norms seconds", time.time() - t3, flush=True)
    out["A_fro"] = np.sqrt(a2.sum())
    out["err_fro"] = np.sqrt(e2.sum())          # exact ||A - A_hat_ref||_F
    out["err_pair"] = np.sqrt(e2)                # (b, b) per-pair exact error norms
    if name == "c4":
        out["sens_fro"] = np.sqrt(d2.sum())      # exact ||A_hat_ref - A_hat_ref(coords + 1 ulp)||_F
        out["sens_pair"] = np.sqrt(d2)
        out["err_fro_pert"] = np.sqrt(f2.sum())  # the perturbed reference's exact error (against the unperturbed A)
        names = ["base", "+1ulp"] + list(family)
        out["err_family_names"] = np.array(names)
        out["err_family"] = np.array([out["err_fro"], out["err_fro_pert"]] + [family[v] for v in family])
    np.savez_compressed(os.path.join(OUT, f"{name}_{mid}.npz"), **out)
    print(name, "A_fro", out["A_fro"], "err/A", out["err_fro"] / out["A_fro"],
          "sens/A", out.get("sens_fro", np.nan) / out["A_fro"], flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c3"]:
        run(name)
