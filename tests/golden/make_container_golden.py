"""UBLR1 container fixtures written by the UNMODIFIED reference's write_ublr
(ref/container.py:38-58). Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_container_golden.py

Stores, per case, the reference's bytes (`*.ublr`) and the arrays they were
written from (`*_arrays.npz`), so tests can check our writer byte-for-byte
without the reference present. Cases: a 1-D grid (b=8, m=16, k=3, tagging A2)
and a ragged 2-D point cloud (b=16, k=5, type B block nullification).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from ublr import (  # noqa: E402
    DenseOperator, RandomStream, build_tessellation, compress, gaussian, grid_points, random_points, write_ublr,
)

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, rep, coords, b):
    write_ublr(os.path.join(OUT, f"{name}.ublr"), rep)
    pairs = sorted(rep.b_blocks)
    np.savez_compressed(
        os.path.join(OUT, f"{name}_arrays.npz"), coords=coords, b=b, rank=rep.rank,
        ranks=np.asarray(rep.effective_ranks), U=np.concatenate(rep.u_blocks, 0), V=np.concatenate(rep.v_blocks, 0),
        core=rep.core, pairs=np.asarray(pairs), B=np.concatenate([rep.b_blocks[p].ravel() for p in pairs]))


def main():
    pts = grid_points(128, 1)
    tess = build_tessellation(pts, 8)
    A = gaussian(128, 128, RandomStream(3))
    rep, _ = compress(DenseOperator(A), tess, 3, "A2", p=5, stream=RandomStream(1), compute_error=False)
    save("container_grid1d", rep, np.asarray(pts.coords if hasattr(pts, "coords") else pts), 8)

    pts = random_points(300, 2, RandomStream(11))
    tess = build_tessellation(pts, 16)
    A = gaussian(300, 300, RandomStream(4))
    rep, _ = compress(DenseOperator(A), tess, 5, "B1", p=4, stream=RandomStream(2), compute_error=False)
    save("container_cloud2d", rep, np.asarray(pts.coords if hasattr(pts, "coords") else pts), 16)


if __name__ == "__main__":
    main()
