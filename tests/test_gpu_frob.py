"""Exact blockwise Frobenius norms on the device (ublr_frob_error /
ublr_frob_diff) against dense numpy on the same representations: uniform,
ragged and dense-operator problems, and block-row ranges (shards)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2501_05528_b200 as P
from test_gpu_compress import gpu_problem

pytestmark = pytest.mark.gpu


def _dense_pairs(tess, M):
    """(b, b) Frobenius norms of the blocks of a dense matrix (original order)."""
    b = tess.b
    out = np.zeros((b, b))
    for i in range(b):
        for j in range(b):
            out[i, j] = np.linalg.norm(M[np.ix_(tess.blocks[i], tess.blocks[j])])
    return out


@pytest.mark.parametrize("name,k,mid", [("log1k_A2", 10, "A2"), ("rand500_A1", 8, "A1"), ("c1s_A2", 10, "A2"),
                                        ("log1k_B2", 8, "B2")])
def test_frobenius_error_matches_dense(name, k, mid):
    tess, op, A = gpu_problem(name)
    rep, _ = P.compress(op, tess, k, mid, p=4, stream=P.RandomStream(7), compute_error=False)
    Ad = A if A is not None else op.dense()
    H = rep.to_dense()
    fr = P.frobenius_error(op, rep)
    want_e = _dense_pairs(tess, Ad - H)
    want_a = _dense_pairs(tess, Ad)
    np.testing.assert_allclose(np.sqrt(fr.pair2), want_e, rtol=1e-9, atol=1e-13 * np.linalg.norm(Ad))
    np.testing.assert_allclose(np.sqrt(fr.ref2), want_a, rtol=1e-12)
    assert fr.relative == pytest.approx(np.linalg.norm(Ad - H) / np.linalg.norm(Ad), rel=1e-8)
    # deterministic
    fr2 = P.frobenius_error(op, rep)
    assert np.array_equal(fr.pair2, fr2.pair2)
    # a block-row range reproduces the same rows
    b = tess.b
    part = P.frobenius_error(op, rep, b // 3, b // 3 + 3)
    assert np.array_equal(part.pair2, fr.pair2[b // 3:b // 3 + 3])


@pytest.mark.parametrize("name,k", [("log1k_A2", 10), ("rand500_A2", 8)])
def test_frobenius_distance_matches_dense(name, k):
    tess, op, _ = gpu_problem(name)
    r1, _ = P.compress(op, tess, k, "A2", p=4, stream=P.RandomStream(7), compute_error=False)
    r2, _ = P.compress(op, tess, k - 2, "A1", p=4, stream=P.RandomStream(8), compute_error=False)
    D = r1.to_dense() - r2.to_dense()
    fd = P.frobenius_distance(r1, r2)
    np.testing.assert_allclose(np.sqrt(fd.pair2), _dense_pairs(tess, D), rtol=1e-9,
                               atol=1e-14 * np.linalg.norm(r1.to_dense()))
    # the same representation: only the accumulation-order rounding of -x + x remains
    assert P.frobenius_distance(r1, r1).fro <= 1e-14 * np.linalg.norm(r1.to_dense())
