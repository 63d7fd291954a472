"""CPU operators for the oracle — TEST INFRASTRUCTURE ONLY.

* `Dense`: explicit matrix (ref/operators.py:41-52).
* `KernelOp`: row-chunked, multithreaded on-the-fly kernel matrix for the
  BASELINE configs (`-log|x-y|` with diagonal `-log(h/2)`, `1/|x-y|` with
  diagonal `2/h`); the 34 GB c3/c4 matrix is never materialised
  (SURVEY.md §8d, F7).
* `synthetic_factors` / `synthetic_dense`: the exact-rank synthetic operator
  of ref/operators.py:193-235, plus the config-1 variant (far core scaled by
  2^-|i-j|, unit-variance near blocks; BASELINE.json configs[0]).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .ublr_oracle import leading_q, normals

__all__ = ["Dense", "KernelOp", "synthetic_factors", "synthetic_dense", "kernel_block"]


class Dense:
    def __init__(self, matrix):
        self.matrix = np.asarray(matrix, dtype=float)
        self.shape = self.matrix.shape

    def apply(self, X):
        return self.matrix @ X

    def apply_adjoint(self, X):
        return self.matrix.T @ X


def kernel_block(coords, rows, cols, kind, diag):
    """Entries A(rows, cols) of the config kernel matrices."""
    xr = coords[rows]
    xc = coords[cols]
    d2 = np.zeros((len(rows), len(cols)))
    for a in range(coords.shape[1]):
        diff = xr[:, a][:, None] - xc[:, a][None, :]
        d2 += diff * diff
    same = np.asarray(rows)[:, None] == np.asarray(cols)[None, :]
    d2[same] = 1.0
    if kind == "log":
        out = -0.5 * np.log(d2)
    elif kind == "inv":
        out = 1.0 / np.sqrt(d2)
    else:
        raise ValueError(f"unknown kernel {kind!r}")
    out[same] = diag
    return out


def blas_threads(n):
    """Context manager limiting the BLAS thread pool to n threads."""
    from threadpoolctl import threadpool_limits
    return threadpool_limits(limits=n, user_api="blas")


class KernelOp:
    """Symmetric kernel matrix applied in row chunks on a thread pool."""

    def __init__(self, coords, kind, diag, chunk=512, threads=None):
        self.coords = np.ascontiguousarray(coords, dtype=float)
        self.kind = kind
        self.diag = float(diag)
        n = self.coords.shape[0]
        self.shape = (n, n)
        self.chunk = chunk
        self.threads = threads or os.cpu_count() or 1

    def _rows(self, lo, hi, X):
        blk = kernel_block(self.coords, np.arange(lo, hi), np.arange(self.shape[0]),
                           self.kind, self.diag)
        return blk @ X

    def apply(self, X):
        X = np.asarray(X, dtype=float)
        n = self.shape[0]
        out = np.empty((n, X.shape[1]))
        spans = [(lo, min(lo + self.chunk, n)) for lo in range(0, n, self.chunk)]
        # one BLAS thread per chunk worker: the pool already occupies every
        # core (nested BLAS threading would oversubscribe them)
        with blas_threads(1), ThreadPoolExecutor(self.threads) as ex:
            for (lo, hi), res in zip(spans, ex.map(lambda s: self._rows(s[0], s[1], X), spans)):
                out[lo:hi] = res
        return out

    apply_adjoint = apply

    def dense(self):
        n = self.shape[0]
        return kernel_block(self.coords, np.arange(n), np.arange(n), self.kind, self.diag)


def synthetic_factors(bx, rank, stream, far_decay=False, near_unit=False):
    """Exact-rank factors (ref/operators.py:193-224). With `far_decay` the far
    core blocks are scaled by 2^-|i-j| and with `near_unit` the near blocks
    keep unit variance (BASELINE config 1); otherwise the reference's scaling
    rank/sqrt(m_i m_j) applies."""
    sizes = bx.sizes
    if rank > sizes.min():
        raise ValueError(f"rank {rank} exceeds smallest block size {sizes.min()}")
    U = [leading_q(normals(sizes[i], rank, stream.child(0, i)), rank) for i in range(bx.b)]
    V = [leading_q(normals(sizes[i], rank, stream.child(1, i)), rank) for i in range(bx.b)]
    core, near = {}, {}
    for i in range(bx.b):
        for j in bx.far(i):
            c = normals(rank, rank, stream.child(2, i * bx.b + j))
            core[(i, j)] = c * 2.0 ** (-abs(i - j)) if far_decay else c
        for j in bx.nbrs[i]:
            g = normals(sizes[i], sizes[j], stream.child(3, i * bx.b + j))
            near[(i, j)] = g if near_unit else (max(rank, 1) / np.sqrt(sizes[i] * sizes[j])) * g
    return U, V, core, near


def synthetic_dense(bx, U, V, core, near):
    """ref/operators.py:227-239."""
    A = np.zeros((bx.n, bx.n))
    for (i, j), c in core.items():
        A[np.ix_(bx.blocks[i], bx.blocks[j])] = U[i] @ c @ V[j].T
    for (i, j), g in near.items():
        A[np.ix_(bx.blocks[i], bx.blocks[j])] = g
    return A
