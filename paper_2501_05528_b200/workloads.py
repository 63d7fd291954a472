"""The BASELINE.json configurations as concrete synthetic inputs.

Input synthesis only (host numpy, outside every timed region); the
compression itself runs on the GPU. See SURVEY.md §8(d) and DESIGN.md.

  c1: d=1, N=2048, b=32, m=64, k=10, p=5, A2, dense synthetic uBLR matrix
  c2: d=2, 64x64 grid (N=4096), b=64, m=64, -log|x-y| (diag -log(h/2)), k=20, p=10, A2
  c3: d=2, 256x256 grid (N=65536), b=256, m=256, same kernel, k=40, p=10, A1
  c4: as c3, B2, k=40 (assumed; BASELINE does not state k), p=10
  c5: d=2, 1024x1024 grid, b=4096, m=256, 1/|x-y| (diag 2/h, assumed), k=48, p=16, A2
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .linalg import RandomStream, gaussian
from .operators import DenseOperator, KernelOperator
from .tessellation import build_tessellation, grid_points

DATA_SEED = 1       # c1 factors: RandomStream(1).child(17) (tests/conftest.py:30 layout)
COMPRESS_SEED = 7   # compression stream RandomStream(7)


@dataclass
class Workload:
    name: str
    tess: object
    op: object
    k: int
    p: int
    method: str
    d: int
    n: int
    b: int
    m: int
    kernel: str
    points: object = None
    matrix: np.ndarray | None = None

    @property
    def ell(self):
        return 3 ** self.d + 1

    def describe(self) -> dict:
        return {"workload": self.name, "N": self.n, "b": self.b, "m": self.m, "k": self.k, "p": self.p,
                "d": self.d, "method": self.method, "operator": self.kernel,
                "seed": COMPRESS_SEED}


def c1_matrix(tess, rank, stream):
    """Config-1 synthetic: far A_ij = U_i (2^-|i-j| G_ij) V_j^T with U_i, V_j the
    leading Q of seeded Gaussians; near blocks unit Gaussians. Factor streams
    follow ref/operators.py:193-224."""
    sizes = tess.block_sizes

    def lq(M):
        return np.linalg.qr(M)[0][:, :rank]

    U = [lq(gaussian(sizes[i], rank, stream.child(0, i))) for i in range(tess.b)]
    V = [lq(gaussian(sizes[i], rank, stream.child(1, i))) for i in range(tess.b)]
    A = np.zeros((tess.n_points, tess.n_points))
    for i in range(tess.b):
        for j in tess.far_fields[i]:
            c = gaussian(rank, rank, stream.child(2, i * tess.b + j)) * 2.0 ** (-abs(i - j))
            A[np.ix_(tess.blocks[i], tess.blocks[j])] = U[i] @ c @ V[j].T
        for j in tess.neighbor_lists[i]:
            A[np.ix_(tess.blocks[i], tess.blocks[j])] = gaussian(sizes[i], sizes[j], stream.child(3, i * tess.b + j))
    return A


def build(name: str, device_ops: bool = True) -> Workload:
    name = name.lower()
    if name == "c1":
        pts = grid_points(2048, 1)
        tess = build_tessellation(pts, 32)
        A = c1_matrix(tess, 10, RandomStream(DATA_SEED).child(17))
        op = DenseOperator(A) if device_ops else None
        return Workload("c1", tess, op, 10, 5, "A2", 1, 2048, 32, 64, "dense-synthetic", pts, A)
    if name in ("c2", "c3", "c4"):
        per, b = (64, 64) if name == "c2" else (256, 256)
        pts = grid_points(per, 2)
        tess = build_tessellation(pts, b)
        op = KernelOperator(pts, "log", -np.log(0.5 / per)) if device_ops else None
        k, p, method = {"c2": (20, 10, "A2"), "c3": (40, 10, "A1"), "c4": (40, 10, "B2")}[name]
        return Workload(name, tess, op, k, p, method, 2, per * per, b, (per * per) // b, "-log|x-y|", pts)
    if name == "c5":
        pts = grid_points(1024, 2)
        tess = build_tessellation(pts, 4096)
        op = KernelOperator(pts, "inv", 2.0 * 1024) if device_ops else None
        return Workload("c5", tess, op, 48, 16, "A2", 2, 1024 * 1024, 4096, 256, "1/|x-y|", pts)
    raise ValueError(f"unknown workload {name!r}")


def algorithmic_flops(w: Workload) -> dict:
    """Algorithmic FP64 flop counts of the kernels for one compression
    (restructured counts where the kernel restructures)."""
    N, b, m, k, p, ell = w.n, w.b, w.m, w.k, w.p, w.ell
    out = {}
    if w.method == "A2":
        gc = k + p
        sides = 2
        # Kronecker-restructured tagged sketch: 2 N^2 gc per side + ell scatter
        out["sketch"] = sides * (2.0 * N * N * gc + 2.0 * N * b * gc * ell)
        out["sketch_dense_equiv"] = sides * 2.0 * N * N * ell * gc
        K = b * min(k, m)
        out["coupling"] = 2.0 * N * N * k + 2.0 * N * K * k
        n_pairs = sum(len(x) for x in w.tess.neighbor_lists)
        out["nearfield"] = 2.0 * b * b * k * k * m / 9.0 * 9 + N * N + n_pairs * 2.0 * m * m * k
    return out
