"""CPU-only tests: host planning, geometry, the C-ABI export table and the
host build of the RNG decode (no compute calls need a GPU here)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import _lib
from cases import golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ublr_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\*]+\s+\**(ublr_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from _lib.SIGNATURES"
    assert lib.ublr_version() == 1


def test_struct_layouts():
    assert C.sizeof(_lib.OpDesc) == 64
    assert C.sizeof(_lib.RngStreamDesc) == 56


@pytest.mark.parametrize("name", ["grid2d", "grid1d", "rand2d", "grid3d"])
def test_tessellation_matches_reference(name):
    g = golden("geometry")
    pts = P.PointCloud(g[f"{name}_coords"], g[f"{name}_coords"].shape[1])
    t = P.build_tessellation(pts, int(g[f"{name}_b"]))
    assert np.array_equal(np.concatenate(t.blocks), g[f"{name}_perm"])
    assert np.array_equal(t.block_sizes, g[f"{name}_sizes"])
    assert np.array_equal(np.concatenate([np.array(x) for x in t.neighbor_lists]), g[f"{name}_nbrflat"])
    assert np.array_equal(P.color_boxes(t).colors, g[f"{name}_colours"])


def test_tagging_plan_bitwise():
    g = golden("plans")
    t = P.build_tessellation(P.grid_points(64, 2), 64)
    plan = P.plan_tagging(t, 0, "gaussian", P.RandomStream(7).child(1))
    assert np.array_equal(plan.matrix.entries, g["c2_T"])
    # null vectors come from the C-ABI Householder (LAPACK convention): equal
    # to the reference's numpy QR up to rounding, same signs
    assert np.abs(plan.Z - g["c2_Z"]).max() <= 1e-14
    assert np.array_equal(np.sign(plan.Z), np.sign(g["c2_Z"]))
    assert np.allclose(plan.rho_base, g["c2_rho"], rtol=1e-10, equal_nan=True)
    t16 = P.build_tessellation(P.grid_points(32, 2), 16)
    plan = P.plan_tagging(t16, 0, "gaussian", P.RandomStream(7).child(1),
                          extra_check=lambda T: P.b2_denominators_ok(T, t16))
    assert np.abs(plan.Z - g["b2s_Z"]).max() <= 1e-14


def test_null_vectors_c_abi_match_numpy():
    """ublr_null_vectors against numpy's complete QR on random row sets of
    every size below ell (the boundary blocks take a specific vector of a
    multi-dimensional null space, so the Householder convention matters)."""
    from paper_2501_05528_b200.tagging import batched_null_vectors, batched_null_vectors_numpy
    rng = np.random.default_rng(3)
    for ell in (5, 10, 28):
        T = rng.standard_normal((40, ell))
        sets = [sorted(rng.choice(40, size=sz, replace=False).tolist()) for sz in range(0, ell) for _ in range(3)]
        Zc, rc, okc = batched_null_vectors(T, sets)
        Zn, rn, okn = batched_null_vectors_numpy(T, sets)
        assert np.abs(Zc - Zn).max() <= 1e-13
        assert okc.all() and okn.all()


def test_pair_vectors_match_oracle():
    import oracle as O
    from paper_2501_05528_b200.tagging import pair_vectors
    t = P.build_tessellation(P.grid_points(32, 2), 16)
    T = P.RandomStream(3).normal(16, 10)
    Z, den = pair_vectors(T, t)
    bx = O.partition(O.cell_centres(32, 2), 16)
    lim = 1e-10 * max(1.0, np.linalg.norm(T))
    p = 0
    for i in range(16):
        for j in bx.nbrs[i]:
            z, d = O.pair_vector(T, bx.nbrs[i], j, lim)
            assert np.abs(z - Z[p]).max() <= 1e-14 and d == pytest.approx(den[p], rel=1e-13)
            p += 1


@pytest.fixture(scope="module")
def rng_host():
    path = os.path.join(ROOT, "tests", "native", "librng_host.so")
    if not os.path.exists(path):
        pytest.skip("tests/native/librng_host.so not built")
    lib = C.CDLL(path)
    lib.host_philox_words.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_void_p]
    lib.host_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_void_p]
    lib.host_normals.restype = C.c_int64
    lib.host_log1p.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
    lib.host_libm_log1p.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
    return lib


def test_log1p_restatement_matches_host_libm(rng_host):
    """csrc/philox_zig.cuh log1p_host_exact (the ziggurat tail's log1p, shared
    by the device decode) against the host C library's log1p — what numpy's
    ziggurat calls through npy_log1p (numpy's log1p ufunc is a different,
    vectorised implementation) — over the tail's argument range -u,
    u in [0, 1), and beyond."""
    rng = np.random.default_rng(3)
    u = (rng.integers(0, 2 ** 53, 4_000_000, dtype=np.uint64) >> np.uint64(0)).astype(np.float64) * 2.0 ** -53
    xs = [-u, np.ldexp(rng.random(200_000), -rng.integers(1, 60, 200_000)),
          -np.ldexp(rng.random(200_000), -rng.integers(1, 60, 200_000)), rng.random(100_000) * 1e6,
          np.array([0.0, -0.0, 2.0 ** -60, -2.0 ** -40, 0.4142, -0.2929, 1e300])]
    for x in xs:
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        want = np.empty_like(x)
        rng_host.host_log1p(x.ctypes.data, x.size, out.ctypes.data)
        rng_host.host_libm_log1p(x.ctypes.data, x.size, want.ctypes.data)
        assert np.array_equal(out, want)


def test_philox_words_match_numpy(rng_host):
    for seed, key in ((7, (0, 0, 3)), (1, ()), (123456789, (2,))):
        st = P.RandomStream(seed, key)
        k0, k1 = st.philox_key()
        bg = np.random.Philox(np.random.SeedSequence(seed, spawn_key=key))
        want = bg.random_raw(1001)
        got = np.zeros(1001, dtype=np.uint64)
        rng_host.host_philox_words(k0, k1, 1001, got.ctypes.data)
        assert np.array_equal(got, want)


def test_ziggurat_decode_matches_numpy(rng_host):
    g = golden("rng")
    for t in range(7):
        spec = g[f"spec{t}"]
        seed, r, c = int(spec[0]), int(spec[1]), int(spec[2])
        key = tuple(int(v) for v in spec[3:] if v >= 0)
        k0, k1 = P.RandomStream(seed, key).philox_key()
        out = np.zeros(r * c)
        rng_host.host_normals(k0, k1, r * c, out.ctypes.data)
        assert np.array_equal(out.reshape(r, c), g[f"normals{t}"])
    # a long stream exercises the wedge and tail branches many times
    st = P.RandomStream(11, (5,))
    k0, k1 = st.philox_key()
    n = 2_000_000
    out = np.zeros(n)
    used = rng_host.host_normals(k0, k1, n, out.ctypes.data)
    want = st.normal(1, n).ravel()
    assert np.array_equal(out, want)
    assert n < used < 1.03 * n


def test_vectorised_seedsequence_matches_numpy():
    from paper_2501_05528_b200.seedseq import philox_keys
    keys = [(0, 0, i) for i in range(200)] + [(0, 1, i) for i in range(200)]
    odd = [(), (0,), (2,), (9, 0), (1, 17, 3), (0, 0, 2 ** 33 + 5), (1, 2 ** 40)]
    for seed in (7, 0, 1, 123456789, 2 ** 40 + 3):
        for ks in (keys, odd, keys[:1]):
            got = philox_keys(seed, ks)
            want = np.array([np.random.SeedSequence(seed, spawn_key=k).generate_state(2, np.uint64) for k in ks])
            assert np.array_equal(got, want)


def test_seedseq_keys_c_abi_matches_numpy():
    """The C-ABI host key derivation (product path) against numpy's SeedSequence."""
    from paper_2501_05528_b200.seedseq import philox_keys_suffixed
    suf = np.array([(s, i) for s in (0, 1) for i in range(300)], dtype=np.int64)
    for seed, prefix in ((7, (0,)), (0, ()), (123456789, (3, 1)), (2 ** 40 + 3, (0, 2 ** 33 + 5)), (5, (0, 0, 9))):
        got = philox_keys_suffixed(seed, prefix, suf)
        want = np.array([np.random.SeedSequence(seed, spawn_key=tuple(prefix) + tuple(int(x) for x in k))
                         .generate_state(2, np.uint64) for k in suf])
        assert np.array_equal(got, want)
    # no spawn key at all
    got = philox_keys_suffixed(11, (), np.zeros((1, 0), dtype=np.int64))
    assert np.array_equal(got[0], np.random.SeedSequence(11).generate_state(2, np.uint64))


def test_quantile_restatement_matches_numpy():
    from paper_2501_05528_b200.reconstruction import _quantiles
    rng = np.random.default_rng(0)
    for n in list(range(1, 30)) + [64, 255, 4096]:
        x = np.sort(rng.standard_normal(n) * rng.uniform(0.1, 1e6))
        assert np.array_equal(np.array(_quantiles(x, (0.25, 0.5, 0.75))), np.quantile(x, (0.25, 0.5, 0.75)))


@pytest.mark.parametrize("per,nb,d", [(64, 64, 2), (16, 64, 3), (48, 16, 2)])
def test_plan_evaluation_c_abi_matches_numpy(per, nb, d):
    """ublr_tag_plan_host (null vectors, residuals, aspect ratios in C) against
    the numpy form of the same evaluation."""
    from paper_2501_05528_b200.tagging import _evaluate, _evaluate_numpy, make_tagging_matrix
    tess = P.build_tessellation(P.grid_points(per, d), nb)
    T = make_tagging_matrix(tess.b, d, 0, "gaussian", P.RandomStream(5).child(1).child(0))
    a, b = _evaluate(T, tess, 1), _evaluate_numpy(T, tess, 1)
    assert np.allclose(np.abs(a.null_vectors.Z), np.abs(b.null_vectors.Z), rtol=0, atol=1e-13)
    assert np.allclose(a.rho_base, b.rho_base, rtol=1e-12, equal_nan=True)


# name -> (per_axis, b, extra_cols, distribution, optimize); tests/golden/make_golden_options.py
PLAN_OPTIONS = {
    "g16_opt": (32, 16, 0, "gaussian", True),
    "g64_opt": (64, 64, 0, "gaussian", True),
    "g16_x2_opt": (32, 16, 2, "gaussian", True),
    "g16_equi": (32, 16, 0, "equidistributed", False),
    "g16_haar_x1": (32, 16, 1, "haar", False),
}


@pytest.mark.parametrize("name", sorted(PLAN_OPTIONS))
def test_tagging_plan_options_match_reference(name):
    """Null-vector optimisation (ref/tagging.py:194-289), equidistributed and
    haar rows (ref/tagging.py:61-123), extra columns, and the extra_samples
    combination vectors (ref/bases.py:177-182) against the reference's plans."""
    per, b, xc, dist, opt = PLAN_OPTIONS[name]
    g = golden("plans_options")
    t = P.build_tessellation(P.grid_points(per, 2), b)
    plan = P.plan_tagging(t, xc, dist, P.RandomStream(7).child(1), optimize=opt)
    assert int(g[f"{name}_attempts"]) == plan.attempts
    T = plan.matrix.entries
    if dist == "gaussian":
        assert np.array_equal(T, g[f"{name}_T"])
    else:   # numpy QR / Riesz descent: the same operations, rounding-level agreement
        assert np.abs(T - g[f"{name}_T"]).max() <= 1e-13
    assert np.abs(plan.Z - g[f"{name}_Z"]).max() <= 1e-10
    assert np.allclose(plan.rho_base, g[f"{name}_rho"], rtol=1e-8, equal_nan=True)
    if opt:
        assert np.allclose(plan.rho_optimized, g[f"{name}_rho_opt"], rtol=1e-8, equal_nan=True)
        fin = ~np.isnan(plan.rho_base)
        assert (plan.rho_optimized[fin] <= plan.rho_base[fin] * (1 + 1e-12)).all()
    else:
        assert plan.rho_optimized is None
    X = P.tagging.extra_sample_vectors(plan, t)
    assert np.abs(X - g[f"{name}_X"]).max() <= 1e-10


def test_optimize_nullity_one_warns_and_keeps_base():
    t = P.build_tessellation(P.grid_points(32, 2), 16)
    plan = P.plan_tagging(t, 0, "gaussian", P.RandomStream(7).child(1))
    interior = next(i for i, nb in enumerate(t.neighbor_lists) if len(nb) == 9)
    base = plan.null_vectors[interior]
    with pytest.warns(UserWarning, match="one-dimensional"):
        nv = P.tagging.optimize_null_vector(plan.matrix, t, interior)
    assert np.abs(nv.vector - base.vector).max() <= 1e-14
