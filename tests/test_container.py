"""UBLR1 container (ref/container.py): byte-for-byte against files written by
the unmodified reference (tests/golden/make_container_golden.py), determinism,
header fields, magic validation; device round trip on the GPU."""

import os

import numpy as np
import pytest

import paper_2501_05528_b200 as P
from paper_2501_05528_b200.container import write_ublr_host

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["container_grid1d", "container_cloud2d"]


def _case(name):
    g = np.load(os.path.join(GOLD, f"{name}_arrays.npz"))
    coords = g["coords"]
    d = coords.shape[1] if coords.ndim == 2 else 1
    tess = P.build_tessellation(P.PointCloud(coords.reshape(len(coords), d), d), int(g["b"]))
    sizes, ranks = tess.block_sizes, g["ranks"]
    cut = np.cumsum(sizes * ranks)[:-1]
    U = [u.reshape(m, r) for u, m, r in zip(np.split(g["U"].ravel(), cut), sizes, ranks)]
    V = [v.reshape(m, r) for v, m, r in zip(np.split(g["V"].ravel(), cut), sizes, ranks)]
    pairs = [tuple(int(x) for x in p) for p in g["pairs"]]
    bcut = np.cumsum([sizes[i] * sizes[j] for i, j in pairs])[:-1]
    B = {p: blk.reshape(sizes[p[0]], sizes[p[1]]) for p, blk in zip(pairs, np.split(g["B"], bcut))}
    return tess, int(g["rank"]), ranks, U, V, g["core"], B


@pytest.mark.parametrize("name", CASES)
def test_host_writer_matches_reference_bytes(name, tmp_path):
    tess, k, ranks, U, V, core, B = _case(name)
    path = tmp_path / "ours.ublr"
    write_ublr_host(path, tess, k, ranks, U, V, core, B)
    ref = open(os.path.join(GOLD, f"{name}.ublr"), "rb").read()
    assert path.read_bytes() == ref


@pytest.mark.parametrize("name", CASES)
def test_header_and_determinism(name, tmp_path):
    tess, k, ranks, U, V, core, B = _case(name)
    p1, p2 = tmp_path / "a.ublr", tmp_path / "b.ublr"
    write_ublr_host(p1, tess, k, ranks, U, V, core, B)
    write_ublr_host(p2, tess, k, ranks, U, V, core, B)
    raw = p1.read_bytes()
    assert raw == p2.read_bytes()
    assert raw[:5] == b"UBLR1"
    h = np.frombuffer(raw, dtype="<u8", count=6, offset=5)
    assert list(h[:4]) == [tess.n_points, tess.b, k, tess.dim]
    assert h[5] == len(B)


def test_magic_validation(tmp_path):
    path = tmp_path / "junk.ublr"
    path.write_bytes(b"NOTUBLR" + b"\x00" * 64)
    with pytest.raises(ValueError):
        P.read_ublr(path)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_round_trip(name, tmp_path):
    """read (reference bytes) -> device UniformBLR -> streamed write: identical
    bytes; the read representation applies like the stored arrays."""
    ref = os.path.join(GOLD, f"{name}.ublr")
    rep = P.read_ublr(ref)
    out = tmp_path / "rt.ublr"
    P.write_ublr(out, rep)
    assert out.read_bytes() == open(ref, "rb").read()
    tess, k, ranks, U, V, core, B = _case(name)
    X = np.random.default_rng(3).standard_normal((tess.n_points, 3))
    roff = np.concatenate(([0], np.cumsum(ranks)))
    want = np.zeros_like(X)
    for i, bi in enumerate(tess.blocks):
        for j, bj in enumerate(tess.blocks):
            blk = U[i] @ core[roff[i]:roff[i + 1], roff[j]:roff[j + 1]] @ V[j].T
            if (i, j) in B:
                blk = blk + B[(i, j)]
            want[bi] += blk @ X[bj]
    assert np.abs(rep.apply(X) - want).max() <= 1e-12 * np.abs(want).max()
