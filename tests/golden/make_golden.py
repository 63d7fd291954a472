"""Generate the golden fixtures by running the UNMODIFIED reference package.

Run in the build container (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Each fixture stores the reference's inputs (seeds/geometry) and outputs for a
small case. Large outputs are stored as fixed random "probes" (block @ w) so
the files stay small while still pinning every entry to rounding.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import ublr  # noqa: E402
from ublr import (  # noqa: E402
    DenseOperator, RandomStream, build_tessellation, color_boxes, compress,
    gaussian, grid_points, laplace2d_operator, plan_tagging, random_points,
)
from ublr.linalg import col_basis  # noqa: E402
from ublr.reconstruction import b2_denominators_ok  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def probe_vec(n, salt):
    return np.random.default_rng(1000 + salt).standard_normal(n)


def c1_matrix(tess, rank, stream):
    """Config-1 synthetic: far blocks U_i (2^-|i-j| G) V_j^T, unit Gaussian
    near blocks (BASELINE.json configs[0]); factor streams as in
    ref/operators.py:193-224."""
    sizes = tess.block_sizes
    U = [col_basis(gaussian(sizes[i], rank, stream.child(0, i)), rank) for i in range(tess.b)]
    V = [col_basis(gaussian(sizes[i], rank, stream.child(1, i)), rank) for i in range(tess.b)]
    A = np.zeros((tess.n_points, tess.n_points))
    for i in range(tess.b):
        for j in tess.far_fields[i]:
            c = gaussian(rank, rank, stream.child(2, i * tess.b + j)) * 2.0 ** (-abs(i - j))
            A[np.ix_(tess.blocks[i], tess.blocks[j])] = U[i] @ c @ V[j].T
        for j in tess.neighbor_lists[i]:
            A[np.ix_(tess.blocks[i], tess.blocks[j])] = gaussian(
                sizes[i], sizes[j], stream.child(3, i * tess.b + j))
    return A


def log_matrix(points, h):
    """-log|x-y| with diagonal -log(h/2) (BASELINE configs 2-4)."""
    A = -laplace2d_operator(points).matrix
    np.fill_diagonal(A, -np.log(h / 2.0))
    return A


def save_rep(name, rep, report, A, extra=None):
    tess = rep.tess
    out = {
        "N": tess.n_points, "b": tess.b, "k": rep.rank,
        "ranks": rep.effective_ranks,
        "U": np.concatenate(rep.u_blocks, axis=0) if rep.u_blocks[0].size else np.zeros((0,)),
        "V": np.concatenate(rep.v_blocks, axis=0) if rep.v_blocks[0].size else np.zeros((0,)),
        "rel_error": report.relative_error if report.relative_error is not None else np.nan,
        "storage_entries": report.storage_entries,
        "matvecs": np.array([[report.matvecs.get(p, {"A": 0})["A"],
                              report.matvecs.get(p, {"Astar": 0})["Astar"]]
                             for p in ("I", "II", "III")]),
        "A_fro": np.linalg.norm(A),
    }
    K = rep.core.shape[0]
    if K * K <= 200_000:
        out["core"] = rep.core
    wk = probe_vec(K, 1)
    out["core_w"] = rep.core @ wk
    out["core_tw"] = rep.core.T @ wk
    pairs = sorted(rep.b_blocks)
    out["pairs"] = np.array(pairs, dtype=np.int64)
    # ragged-safe: probes of all pairs concatenated in sorted pair order
    out["B_w"] = np.concatenate([rep.b_blocks[p] @ probe_vec(rep.b_blocks[p].shape[1], 2) for p in pairs])
    out["B_tw"] = np.concatenate([rep.b_blocks[p].T @ probe_vec(rep.b_blocks[p].shape[0], 3) for p in pairs])
    out["B_fro"] = np.array([np.linalg.norm(rep.b_blocks[p]) for p in pairs])
    # full assembled-operator probe: A_hat @ W for a fixed 3-column W
    W = np.stack([probe_vec(tess.n_points, 10 + c) for c in range(3)], axis=1)
    out["Ahat_W"] = rep.apply(W)
    out["Ahat_tW"] = rep.apply_adjoint(W)
    out["err_fro"] = np.linalg.norm(A - rep.to_dense()) / np.linalg.norm(A) if tess.n_points <= 4096 else np.nan
    if extra:
        out.update(extra)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print(name, {k: (v.shape if hasattr(v, "shape") else v) for k, v in out.items()})


def main():
    # --- RNG: Philox keys and normals of several streams --------------------
    cases = [(7, (0, 0, 0), 64, 15), (7, (0, 0, 3), 64, 15), (7, (0, 1, 31), 64, 15),
             (7, (0, 0), 50, 37), (1, (17, 2, 5), 10, 10), (123456789, (), 7, 300),
             (7, (0, 0, 1), 256, 266)]
    rng = {}
    for t, (seed, key, r, c) in enumerate(cases):
        ss = np.random.SeedSequence(seed, spawn_key=key)
        rng[f"key{t}"] = ss.generate_state(2, np.uint64)
        st = RandomStream(seed)
        st = st.child(*key) if key else st
        rng[f"normals{t}"] = st.normal(r, c)
        rng[f"spec{t}"] = np.array([seed, r, c] + list(key) + [-1] * (4 - len(key)), dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **rng)

    # --- geometry ------------------------------------------------------------
    geo = {}
    for name, pts, b in (("grid2d", grid_points(16, 2), 16), ("grid1d", grid_points(64, 1), 8),
                         ("rand2d", random_points(500, 2, RandomStream(21)), 16),
                         ("grid3d", grid_points(8, 3), 8)):
        tess = build_tessellation(pts, b)
        geo[f"{name}_coords"] = pts.coords
        geo[f"{name}_b"] = np.array(b)
        geo[f"{name}_perm"] = np.concatenate(tess.blocks)
        geo[f"{name}_sizes"] = tess.block_sizes
        geo[f"{name}_nbrs"] = np.array([len(x) for x in tess.neighbor_lists])
        geo[f"{name}_nbrflat"] = np.concatenate([np.array(x) for x in tess.neighbor_lists])
        geo[f"{name}_colours"] = np.asarray(color_boxes(tess).colors)
        geo[f"{name}_grid"] = tess.grid_coords
    np.savez_compressed(os.path.join(OUT, "geometry.npz"), **geo)

    # --- tagging plans -------------------------------------------------------
    plans = {}
    tess = build_tessellation(grid_points(64, 2), 64)
    plan = plan_tagging(tess, 0, "gaussian", RandomStream(7).child(1))
    plans["c2_T"] = plan.matrix.entries
    plans["c2_Z"] = np.stack([nv.vector for nv in plan.null_vectors])
    plans["c2_rho"] = plan.rho_base
    plans["c2_attempts"] = np.array(plan.attempts)
    tess16 = build_tessellation(grid_points(32, 2), 16)
    plan = plan_tagging(tess16, 0, "gaussian", RandomStream(7).child(1),
                        extra_check=lambda T: b2_denominators_ok(T, tess16))
    plans["b2s_T"] = plan.matrix.entries
    plans["b2s_Z"] = np.stack([nv.vector for nv in plan.null_vectors])
    plans["b2s_attempts"] = np.array(plan.attempts)
    np.savez_compressed(os.path.join(OUT, "plans.npz"), **plans)

    # --- end-to-end compressions ---------------------------------------------
    # c1s: config-1 style (d=1, m=64, k=10, p=5) at b=8
    tess = build_tessellation(grid_points(512, 1), 8)
    A = c1_matrix(tess, 10, RandomStream(1).child(17))
    rep, report = compress(DenseOperator(A), tess, 10, method_id="A2", p=5, stream=RandomStream(7))
    save_rep("c1s_A2", rep, report, A, {"A_sum": A.sum(), "A_w": A @ probe_vec(512, 4)})

    # full config 1 (N=2048, b=32): core 320x320 stored, B as probes
    tess = build_tessellation(grid_points(2048, 1), 32)
    A = c1_matrix(tess, 10, RandomStream(1).child(17))
    rep, report = compress(DenseOperator(A), tess, 10, method_id="A2", p=5, stream=RandomStream(7))
    save_rep("c1_A2", rep, report, A, {"A_sum": A.sum(), "A_w": A @ probe_vec(2048, 4)})

    # 2D log kernel, 32x32 grid, 16 boxes of 64 points — every method
    pts = grid_points(32, 2)
    tess = build_tessellation(pts, 16)
    A = log_matrix(pts, 1.0 / 32)
    for mid, k, p in (("A2", 10, 5), ("A1", 8, 4), ("A3", 8, 4), ("B1", 8, 4), ("B2", 8, 4)):
        rep, report = compress(DenseOperator(A), tess, k, method_id=mid, p=p, stream=RandomStream(7))
        save_rep(f"log1k_{mid}", rep, report, A)

    # full config 2 (N=4096 log kernel, b=64, k=20, p=10, A2)
    pts = grid_points(64, 2)
    tess = build_tessellation(pts, 64)
    A = log_matrix(pts, 1.0 / 64)
    rep, report = compress(DenseOperator(A), tess, 20, method_id="A2", p=10, stream=RandomStream(7))
    save_rep("c2_A2", rep, report, A)

    # ragged random points (tiny blocks exercise the identity-basis path)
    pts = random_points(500, 2, RandomStream(21))
    tess = build_tessellation(pts, 16)
    A = -laplace2d_operator(pts).matrix
    np.fill_diagonal(A, 3.0)
    for mid in ("A2", "A1", "B2"):
        rep, report = compress(DenseOperator(A), tess, 8, method_id=mid, p=4, stream=RandomStream(9))
        save_rep(f"rand500_{mid}", rep, report, A, {"coords": pts.coords})


if __name__ == "__main__":
    print("reference ublr", ublr.__version__, "numpy", np.__version__)
    main()
