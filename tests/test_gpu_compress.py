"""End-to-end GPU parity: compress() through the CUDA path against the CPU
oracle and the reference's golden fixtures.

Gate (BASELINE.json north_star): ||A_hat_gpu - A_hat_ref||_F / ||A||_F <= 1e-10
and ||A - A_hat_gpu||_F / ||A||_F <= 1.05 x the reference's.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O
import paper_2501_05528_b200 as P
from cases import build_case, golden, probe_vec

pytestmark = pytest.mark.gpu
TOL = 1e-10


def gpu_problem(name):
    """The same input as cases.build_case, as GPU operators."""
    if name.startswith("c1"):
        from cases import c1_problem
        n, b = (512, 8) if name.startswith("c1s") else (2048, 32)
        _, A = c1_problem(n, b)
        tess = P.build_tessellation(P.grid_points(n, 1), b)
        return tess, P.DenseOperator(A), A
    if name.startswith("log1k") or name.startswith("c2"):
        per, b = (32, 16) if name.startswith("log1k") else (64, 64)
        pts = P.grid_points(per, 2)
        tess = P.build_tessellation(pts, b)
        op = P.KernelOperator(pts, "log", -np.log(0.5 / per))
        return tess, op, None
    if name.startswith("rand500"):
        from cases import rand500_problem
        _, coords, _ = rand500_problem()
        tess = P.build_tessellation(P.PointCloud(coords, 2), 16)
        return tess, P.KernelOperator(coords, "log", 3.0), None
    raise KeyError(name)


def ahat_error_vs_golden(rep, g, ncols=3):
    W = np.stack([probe_vec(rep.n, 10 + c) for c in range(ncols)], axis=1)
    scale = float(g["A_fro"])
    e1 = np.linalg.norm(rep.apply(W) - g["Ahat_W"]) / (scale * np.sqrt(ncols))
    e2 = np.linalg.norm(rep.apply_adjoint(W) - g["Ahat_tW"]) / (scale * np.sqrt(ncols))
    return max(e1, e2)


@pytest.mark.parametrize("name", ["c1s_A2", "log1k_A2", "rand500_A2", "c1_A2", "c2_A2",
                                  "log1k_A1", "rand500_A1", "log1k_A3", "log1k_B1", "log1k_B2", "rand500_B2"])
def test_compress_matches_reference(name):
    tess, op, _ = gpu_problem(name)
    _, _, k, p, mid, seed = build_case(name)
    rep, report = P.compress(op, tess, k, mid, p=p, stream=P.RandomStream(seed), compute_error=False)
    g = golden(name)
    assert ahat_error_vs_golden(rep, g) <= TOL
    mv = np.array([[report.matvecs.get(ph, {"A": 0})["A"], report.matvecs.get(ph, {"Astar": 0})["Astar"]]
                   for ph in ("I", "II", "III")])
    assert np.array_equal(mv, g["matvecs"])
    assert report.storage_entries == int(g["storage_entries"])


@pytest.mark.parametrize("name", ["c1s_A2", "log1k_A2", "c2_A2", "log1k_A1", "log1k_A3", "log1k_B1",
                                  "log1k_B2"])
def test_compress_dense_frobenius_vs_oracle(name):
    """Full ||A_hat_gpu - A_hat_oracle||_F / ||A||_F on the same inputs, and the
    approximation error within 1.05x of the oracle's."""
    tess, op, A = gpu_problem(name)
    bx, oop, k, p, mid, seed = build_case(name)
    rep, _ = P.compress(op, tess, k, mid, p=p, stream=P.RandomStream(seed), compute_error=False)
    orep, _ = O.compress(oop, bx, k, mid, p=p, stream=O.Stream(seed), compute_error=False)
    Ad = oop.matrix
    D_gpu, D_ref = rep.to_dense(), orep.to_dense()
    nA = np.linalg.norm(Ad)
    assert np.linalg.norm(D_gpu - D_ref) / nA <= TOL
    err_gpu = np.linalg.norm(Ad - D_gpu) / nA
    err_ref = np.linalg.norm(Ad - D_ref) / nA
    assert err_gpu <= 1.05 * err_ref + 1e-15


@pytest.mark.parametrize("name", ["log1k_A2", "c1s_A2"])
def test_relative_error_estimate_close_to_reference(name):
    """The reference's 20-step power-method estimate, same start vectors."""
    tess, op, _ = gpu_problem(name)
    _, _, k, p, mid, seed = build_case(name)
    rep, report = P.compress(op, tess, k, mid, p=p, stream=P.RandomStream(seed), compute_error=True)
    g = golden(name)
    ref = float(g["rel_error"])
    if ref < 1e-11:   # exact-rank case: both estimates sit at rounding level
        assert report.relative_error < 1e-11
    else:
        assert report.relative_error == pytest.approx(ref, rel=1e-4)


def _uniform_synthetic(d, b, m, k, seed):
    """tests/conftest.py:20-31 of the reference: exact-rank synthetic on a grid."""
    per_axis = round(b ** (1.0 / d))
    pts_axis = per_axis * round(m ** (1.0 / d))
    coords = O.cell_centres(pts_axis, d)
    bx = O.partition(coords, b)
    U, V, core, near = O.synthetic_factors(bx, k, O.Stream(seed).child(17))
    A = O.synthetic_dense(bx, U, V, core, near)
    tess = P.build_tessellation(P.PointCloud(coords, d), b)
    return bx, tess, A


@pytest.mark.parametrize("mid", ["A2", "A3", "B2"])
def test_three_dimensional_geometry(mid):
    """27-neighbour neighbourhoods, 28-column tagging (ref tests/test_reconstruction.py:441-447)."""
    bx, tess, A = _uniform_synthetic(3, 64, 8, 3, 1)
    assert max(len(n) for n in tess.neighbor_lists) == 27
    rep, report = P.compress(P.DenseOperator(A), tess, 3, mid, stream=P.RandomStream(2), compute_error=True)
    assert report.relative_error <= 1e-7
    orep, _ = O.compress(O.Dense(A), bx, 3, mid, p=10, stream=O.Stream(2), compute_error=False)
    assert np.linalg.norm(rep.to_dense() - orep.to_dense()) / np.linalg.norm(A) <= 1e-10


@pytest.mark.parametrize("mid", ["A1", "A2", "A3", "B1", "B2"])
def test_rank_at_least_block_size_uses_identity_bases(mid):
    """k >= m_i: the reference keeps the identity basis (ref/bases.py:78-83)."""
    bx, tess, A = _uniform_synthetic(1, 8, 16, 4, 3)
    k = 16
    rep, _ = P.compress(P.DenseOperator(A), tess, k, mid, p=4, stream=P.RandomStream(4), compute_error=False)
    orep, _ = O.compress(O.Dense(A), bx, k, mid, p=4, stream=O.Stream(4), compute_error=False)
    assert np.array_equal(rep.effective_ranks, orep.ranks)
    assert np.linalg.norm(rep.to_dense() - orep.to_dense()) / np.linalg.norm(A) <= 1e-10


@pytest.mark.parametrize("mid", ["A1", "A2", "A3", "B1", "B2"])
def test_exact_rank_recovery_all_methods(mid):
    """Acceptance criterion 1 of the reference (tests/test_acceptance.py:44-72)."""
    for d, b, m, k in ((1, 8, 16, 2), (1, 8, 40, 5), (2, 16, 16, 2), (2, 81, 16, 5)):
        bx, tess, A = _uniform_synthetic(d, b, m, k, 100 + b)
        _, report = P.compress(P.DenseOperator(A), tess, k, mid, p=10, stream=P.RandomStream(55),
                               error_iterations=20)
        assert report.relative_error <= 1e-7, (d, b, m, k, report.relative_error)


@pytest.mark.parametrize("per,b,kind,k,mid", [(64, 16, "inv", 48, "A2"), (50, 16, "log", 20, "A2"),
                                              (48, 9, "log", 30, "A1"), (50, 16, "log", 20, "B2"),
                                              (50, 16, "log", 16, "B1"), (40, 16, "inv", 12, "B2")])
def test_large_blocks_vs_oracle(per, b, kind, k, mid):
    """m > 64 blocks (the warp-specialised coupling and the v3 near-field
    kernels), uniform m = 256 and ragged 144-169-point blocks, GPU vs the
    oracle's dense compression on the same inputs."""
    pts = P.grid_points(per, 2)
    tess = P.build_tessellation(pts, b)
    diag = -np.log(0.5 / per) if kind == "log" else 2.0 * per
    rep, _ = P.compress(P.KernelOperator(pts, kind, diag), tess, k, mid, p=10, stream=P.RandomStream(5),
                        compute_error=False)
    coords = O.cell_centres(per, 2)
    bx = O.partition(coords, b)
    n = per * per
    A = O.kernel_block(coords, np.arange(n), np.arange(n), kind, diag)
    orep, _ = O.compress(O.Dense(A), bx, k, mid, p=10, stream=O.Stream(5), compute_error=False)
    nA = np.linalg.norm(A)
    D_gpu, D_ref = rep.to_dense(), orep.to_dense()
    assert np.linalg.norm(D_gpu - D_ref) / nA <= TOL
    assert np.linalg.norm(A - D_gpu) / nA <= 1.05 * np.linalg.norm(A - D_ref) / nA + 1e-15


def test_redraw_after_speculative_bases(monkeypatch):
    """The tag pipeline builds bases and queues phases II-III from the device
    draw of the first tagging matrix before the host evaluates the redraw
    policy; when the policy redraws, everything is recomputed for the accepted
    matrix (same result as building from that plan directly) and the ledger
    is not billed twice."""
    import warnings
    import torch
    import paper_2501_05528_b200.reconstruction as R
    from paper_2501_05528_b200.bases import tagging_bases
    pts = P.grid_points(32, 2)
    tess = P.build_tessellation(pts, 16)
    op = P.KernelOperator(pts, "log", -np.log(0.5 / 32))
    _, normal = P.compress(op, tess, 10, "A2", p=5, stream=P.RandomStream(7), compute_error=False)
    orig = R.plan_tagging
    monkeypatch.setattr(R, "plan_tagging", lambda *a, **kw: orig(*a, **{**kw, "ratio_limit": 0.0}))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        rep, report = P.compress(op, tess, 10, "A2", p=5, stream=P.RandomStream(7), compute_error=False)
        plan = orig(tess, 0, "gaussian", P.RandomStream(7).child(1), max_redraws=5, ratio_limit=0.0)
    assert report.aspect_ratios["draws"] == 6
    assert report.matvecs == normal.matvecs
    bases, _ = tagging_bases(op, tess, 10, 5, plan, P.RandomStream(7).child(0))
    assert torch.equal(bases.U, rep.U[:, :10]) and torch.equal(bases.V, rep.V[:, :10])
    core = R.direct_core(op, tess, bases)
    assert torch.equal(core, rep.core_d)


# tests/golden/make_golden_options.py: the 32 x 32 log grid, 16 boxes
OPTION_CASES = {
    "A2_opt": ("A2", 10, 5, {"optimize": True}),
    "A2_xs": ("A2", 10, 5, {"extra_samples": True}),
    "A2_equi": ("A2", 10, 5, {"distribution": "equidistributed"}),
    "A2_haar_x1": ("A2", 10, 5, {"distribution": "haar", "extra_cols": 1}),
    "A2_x2_opt": ("A2", 10, 5, {"extra_cols": 2, "optimize": True}),
    "B2_opt": ("B2", 8, 4, {"optimize": True}),
}


@pytest.mark.parametrize("name", sorted(OPTION_CASES))
def test_tagging_options_match_reference(name):
    """Null-vector optimisation, extra_samples, equidistributed / haar rows and
    extra tagging columns through the GPU path against the reference's own
    compressions of the same matrix (same seeds)."""
    mid, k, p, kw = OPTION_CASES[name]
    tess, op, _ = gpu_problem("log1k_" + mid)
    rep, report = P.compress(op, tess, k, mid, p=p, stream=P.RandomStream(7), compute_error=False, **kw)
    g = golden("opt_" + name)
    assert ahat_error_vs_golden(rep, g) <= TOL
    mv = np.array([[report.matvecs.get(ph, {"A": 0})["A"], report.matvecs.get(ph, {"Astar": 0})["Astar"]]
                   for ph in ("I", "II", "III")])
    assert np.array_equal(mv, g["matvecs"])
    if kw.get("optimize"):
        assert report.aspect_ratios["optimized"]["max"] == pytest.approx(float(g["rho_opt_max"]), rel=1e-8)


def test_compress_on_a_side_stream_matches_default_stream():
    """The speculative path queues the null vectors on a side stream keyed by
    the caller's stream: a compression issued on a user stream, back to back
    with one on the default stream, gives the same bits."""
    tess, op, _ = gpu_problem("c2_A2")
    _, _, k, p, mid, seed = build_case("c2_A2")
    rep0, _ = P.compress(op, tess, k, mid, p=p, stream=P.RandomStream(seed), compute_error=False)
    h0 = rep0.to_host()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        rep1, _ = P.compress(op, tess, k, mid, p=p, stream=P.RandomStream(seed), compute_error=False)
        h1 = rep1.to_host()
    torch.cuda.synchronize()
    for key in ("U", "V", "core", "B"):
        assert np.array_equal(h0[key], h1[key]), key


class HostMatrixOperator:
    """A plain-Python black-box operator: shape / apply / apply_adjoint on
    numpy arrays only (ref/operators.py:24-35, "any object with..." at
    pkg/README.md:113-115). No device descriptor: every operator product of
    the pipeline goes through these host calls."""

    def __init__(self, A):
        self.A = np.asarray(A, dtype=float)
        self.shape = self.A.shape
        self.calls = 0

    def apply(self, X):
        self.calls += 1
        return self.A @ X

    def apply_adjoint(self, X):
        self.calls += 1
        return self.A.T @ X


@pytest.mark.parametrize("name", ["log1k_A1", "log1k_A2", "log1k_A3", "log1k_B1", "log1k_B2", "rand500_A1",
                                  "rand500_A2", "rand500_B2", "c1s_A2"])
def test_black_box_host_operator_matches_reference(name):
    """Phases I-III with a plain-Python operator (sketch, direct_core through
    op.apply(V_dense), one identity probe per colour) against the reference's
    goldens and ledger."""
    tess, dev_op, A = gpu_problem(name)
    Ad = A if A is not None else dev_op.dense()
    op = HostMatrixOperator(Ad)
    _, _, k, p, mid, seed = build_case(name)
    rep, report = P.compress(op, tess, k, mid, p=p, stream=P.RandomStream(seed), compute_error=True)
    g = golden(name)
    assert ahat_error_vs_golden(rep, g) <= TOL
    mv = np.array([[report.matvecs.get(ph, {"A": 0})["A"], report.matvecs.get(ph, {"Astar": 0})["Astar"]]
                   for ph in ("I", "II", "III")])
    assert np.array_equal(mv, g["matvecs"])
    assert op.calls > 0


def test_custom_colouring_matches_oracle():
    """A caller-supplied valid colouring (not color_boxes) gives the
    reference's colour-probe near field for that colouring (device operator
    and black-box operator alike)."""
    import paper_2501_05528_b200.reconstruction as R
    from paper_2501_05528_b200.bases import tagging_bases
    from paper_2501_05528_b200.tessellation import BoxColoring
    tess, op, _ = gpu_problem("log1k_A2")
    Ad = op.dense()
    # greedy distance-2 colouring in reverse block order: valid, different from color_boxes
    nb = [set(x) for x in tess.neighbor_lists]
    cols = np.full(tess.b, -1)
    for i in reversed(range(tess.b)):
        used = {cols[j] for j in range(tess.b) if cols[j] >= 0 and j != i and nb[i] & nb[j]}
        c = 0
        while c in used:
            c += 1
        cols[i] = c
    assert not np.array_equal(cols, P.color_boxes(tess).colors)
    colouring = BoxColoring(colors=cols, num_colors=int(cols.max()) + 1)
    plan = P.plan_tagging(tess, 0, "gaussian", P.RandomStream(7).child(1))
    bases, _ = tagging_bases(op, tess, 10, 5, plan, P.RandomStream(7).child(0))
    core = R.direct_core(op, tess, bases)
    B_dev = R.structured_identity_discrepancy(op, tess, bases, core, colouring).cpu().numpy()
    B_host = R.structured_identity_discrepancy(HostMatrixOperator(Ad), tess, bases, core, colouring).cpu().numpy()
    # oracle: the reference's probe loop on the same bases and core
    bx = O.partition(O.cell_centres(32, 2), 16)
    dt = bases.dt
    Ub = [bases.U[dt.off_h[i]:dt.off_h[i + 1], :10].cpu().numpy() for i in range(tess.b)]
    Vb = [bases.V[dt.off_h[i]:dt.off_h[i + 1], :10].cpu().numpy() for i in range(tess.b)]
    bs = O.Bases(Ub, Vb, np.full(tess.b, 10), "tag")
    Bref = O.near_colour_probes(O.Dense(Ad), bx, bs, core.cpu().numpy(), cols)
    want = np.concatenate([Bref[(int(i), int(j))].ravel() for i, j in zip(dt.pair_i_h, dt.nidx_h)])
    scale = np.linalg.norm(Ad)
    assert np.linalg.norm(B_dev - want) <= 1e-12 * scale
    assert np.linalg.norm(B_host - want) <= 1e-12 * scale


@pytest.mark.parametrize("per,b,k,mid", [(100, 16, 30, "A2"), (64, 16, 80, "A2"), (50, 16, 70, "A1")])
def test_generic_block_sizes_and_ranks_vs_oracle(per, b, k, mid):
    """Blocks above 256 points (625) and ranks above 64: the general coupling /
    near-field kernels (csrc/coupling_gen.cu), GPU vs the oracle's dense
    compression of the same -log kernel matrix."""
    pts = P.grid_points(per, 2)
    tess = P.build_tessellation(pts, b)
    diag = -np.log(0.5 / per)
    rep, _ = P.compress(P.KernelOperator(pts, "log", diag), tess, k, mid, p=10, stream=P.RandomStream(5),
                        compute_error=False)
    coords = O.cell_centres(per, 2)
    bx = O.partition(coords, b)
    n = per * per
    A = O.kernel_block(coords, np.arange(n), np.arange(n), "log", diag)
    orep, _ = O.compress(O.Dense(A), bx, k, mid, p=10, stream=O.Stream(5), compute_error=False)
    nA = np.linalg.norm(A)
    D_gpu, D_ref = rep.to_dense(), orep.to_dense()
    assert np.linalg.norm(D_gpu - D_ref) / nA <= TOL
    # (k = 70 on 144-169-point blocks is exact to rounding: both errors sit
    # near 1e-15, where the 1.05x ratio is not meaningful; floor 1e-13)
    assert np.linalg.norm(A - D_gpu) / nA <= max(1.05 * np.linalg.norm(A - D_ref) / nA, 1e-13)


def test_paper_scale_suggested_blocks():
    """The paper's own setting: N ~ 100k, k = 30,
    b = suggest_block_count(N, k, d) (ref/tessellation.py:127-140) gives
    169 boxes of 576-625 points. Runs through A2 end to end; the exact
    blockwise Frobenius error is small and the near / far structure holds."""
    per = 316
    n = per * per
    b = P.suggest_block_count(n, 30, 2)
    assert b == 169
    pts = P.grid_points(per, 2)
    tess = P.build_tessellation(pts, b)
    assert tess.max_block_size > 256
    op = P.KernelOperator(pts, "log", -np.log(0.5 / per))
    rep, report = P.compress(op, tess, 30, "A2", p=10, stream=P.RandomStream(7), compute_error=False)
    fr = P.frobenius_error(op, rep)
    print(f"N={n} b={b} m_max={tess.max_block_size}: ||A - A_hat||_F / ||A||_F = {fr.relative:.3e}")
    assert fr.relative < 1e-5
    assert report.matvecs["II"]["A"] == 30 * b
