"""Shared problem definitions for the oracle and GPU parity tests.

Each case mirrors one golden fixture written by tests/golden/make_golden.py.
"""

import os

import numpy as np

import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def c1_problem(n, b, k=10):
    """Config-1 synthetic (d=1): oracle boxes + dense matrix."""
    bx = O.partition(O.cell_centres(n, 1), b)
    U, V, core, near = O.synthetic_factors(bx, k, O.Stream(1).child(17), far_decay=True, near_unit=True)
    return bx, O.synthetic_dense(bx, U, V, core, near)


def log_problem(per_axis, b):
    coords = O.cell_centres(per_axis, 2)
    bx = O.partition(coords, b)
    h = 1.0 / per_axis
    return bx, coords, O.KernelOp(coords, "log", -np.log(h / 2.0))


def rand500_problem():
    coords = O.Stream(21).uniform(500, 2)
    bx = O.partition(coords, 16)
    op = O.KernelOp(coords, "log", 3.0)
    return bx, coords, op


# name -> (builder, k, p, method, seed)
def build_case(name):
    if name == "c1s_A2":
        bx, A = c1_problem(512, 8)
        return bx, O.Dense(A), 10, 5, "A2", 7
    if name == "c1_A2":
        bx, A = c1_problem(2048, 32)
        return bx, O.Dense(A), 10, 5, "A2", 7
    if name.startswith("log1k_"):
        mid = name.split("_")[1]
        bx, _, op = log_problem(32, 16)
        k, p = (10, 5) if mid == "A2" else (8, 4)
        return bx, O.Dense(op.dense()), k, p, mid, 7
    if name == "c2_A2":
        bx, _, op = log_problem(64, 64)
        return bx, O.Dense(op.dense()), 20, 10, "A2", 7
    if name.startswith("rand500_"):
        bx, _, op = rand500_problem()
        return bx, O.Dense(op.dense()), 8, 4, name.split("_")[1], 9
    raise KeyError(name)


def probe_vec(n, salt):
    return np.random.default_rng(1000 + salt).standard_normal(n)


def summarize(bx, U_blocks, V_blocks, core, B, ranks):
    """The same probes make_golden.py stores, from any representation given
    as per-block lists in reference (global) index order."""
    K = core.shape[0]
    wk = probe_vec(K, 1)
    pairs = sorted(B)
    out = {
        "U": np.concatenate(U_blocks, axis=0), "V": np.concatenate(V_blocks, axis=0),
        "core_w": core @ wk, "core_tw": core.T @ wk,
        "pairs": np.array(pairs, dtype=np.int64),
        "B_w": np.concatenate([B[p] @ probe_vec(B[p].shape[1], 2) for p in pairs]),
        "B_tw": np.concatenate([B[p].T @ probe_vec(B[p].shape[0], 3) for p in pairs]),
        "B_fro": np.array([np.linalg.norm(B[p]) for p in pairs]),
        "ranks": np.asarray(ranks),
    }
    if K * K <= 200_000:
        out["core"] = core
    return out
