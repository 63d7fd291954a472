"""GPU parity of the individual CUDA kernels (through the C ABI) against the
CPU oracle / numpy on the same seeded inputs."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O
import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import _lib
from paper_2501_05528_b200.bases import draw_test_blocks, tagged_sketch
from paper_2501_05528_b200.linalg import device_normals
from paper_2501_05528_b200.tessellation import device_tess
from cases import golden

pytestmark = pytest.mark.gpu
DEV = "cuda"


def test_rng_streams_bitwise():
    g = golden("rng")
    specs, want, at = [], [], 0
    for t in range(7):
        spec = g[f"spec{t}"]
        seed, r, c = int(spec[0]), int(spec[1]), int(spec[2])
        key = tuple(int(v) for v in spec[3:] if v >= 0)
        specs.append((P.RandomStream(seed, key), r, c, at, c, None))
        want.append(g[f"normals{t}"].ravel())
        at += r * c
    out = torch.full((at,), np.nan, dtype=torch.float64, device=DEV)
    device_normals(specs, out)
    assert np.array_equal(out.cpu().numpy(), np.concatenate(want))


def test_rng_long_stream_with_rowmap():
    rows, cols = 3000, 777
    st = P.RandomStream(7, (0, 0))
    perm = np.random.default_rng(0).permutation(rows).astype(np.int32)
    rowmap = torch.from_numpy(perm).to(DEV)
    out = torch.empty((rows, cols), dtype=torch.float64, device=DEV)
    device_normals([(st, rows, cols, 0, cols, rowmap)], out)
    want = st.normal(rows, cols)
    got = out.cpu().numpy()[perm]
    # bit for bit, tail samples included (log1p restated as the host libm
    # computes it, csrc/philox_zig.cuh)
    assert np.array_equal(got, want)


def test_rng_many_small_streams():
    b, m, gc = 300, 64, 30
    t = P.build_tessellation(P.grid_points(b * m, 1), b) if False else None
    specs = [(P.RandomStream(7).child(0).child(0, i), m, gc, i * m * gc, gc, None) for i in range(b)]
    out = torch.empty(b * m * gc, dtype=torch.float64, device=DEV)
    device_normals(specs, out)
    got = out.cpu().numpy().reshape(b, m, gc)
    for i in (0, 1, 17, 299):
        assert np.array_equal(got[i], P.RandomStream(7).child(0).child(0, i).normal(m, gc))


@pytest.mark.parametrize("rows,cols", [(1, 1), (7, 3), (50, 30), (64, 30), (100, 50), (256, 266)])
def test_rng_per_cta_decode_bitwise(rows, cols):
    """Short streams take the one-launch per-CTA decode (chunk sizes 8, 16 and
    32 words by stream length); bitwise against numpy for every stream."""
    nst = 9
    specs = [(P.RandomStream(11).child(3, i), rows, cols, i * rows * cols, cols, None) for i in range(nst)]
    out = torch.full((nst * rows * cols,), np.nan, dtype=torch.float64, device=DEV)
    device_normals(specs, out)
    got = out.cpu().numpy().reshape(nst, rows, cols)
    for i in range(nst):
        assert np.array_equal(got[i], P.RandomStream(11).child(3, i).normal(rows, cols)), i


def _dense_apply_case(kind):
    coords = O.cell_centres(24, 2)
    n = len(coords)
    if kind == "dense":
        A = np.random.default_rng(1).standard_normal((n, n))
        return coords, P.DenseOperator(A), A
    diag = 3.25
    op = P.KernelOperator(coords, kind, diag)
    A = O.kernel_block(coords, np.arange(n), np.arange(n), kind, diag)
    return coords, op, A


@pytest.mark.parametrize("kind", ["dense", "log", "inv"])
@pytest.mark.parametrize("w", [1, 37, 200])
def test_apply_matches_numpy(kind, w):
    coords, op, A = _dense_apply_case(kind)
    X = np.random.default_rng(2).standard_normal((A.shape[0], w))
    got = op.apply(X)
    want = A @ X
    assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(A) * np.linalg.norm(X)
    got_t = op.apply_adjoint(X)
    assert np.linalg.norm(got_t - A.T @ X) <= 1e-13 * np.linalg.norm(A) * np.linalg.norm(X)


def test_fast_log_accuracy():
    # kernel entries through the apply kernel with unit vectors
    coords = np.random.default_rng(5).uniform(size=(300, 2))
    op = P.KernelOperator(coords, "log", 0.0)
    A = O.kernel_block(coords, np.arange(300), np.arange(300), "log", 0.0)
    got = op.apply(np.eye(300))
    err = np.abs(got - A)
    assert err.max() <= 4e-16 * max(1.0, np.abs(A).max()) * 8


@pytest.mark.parametrize("case", ["c1s", "log1k", "rand500", "inv1k", "inv_rand500", "inv3d"])
def test_tagged_sketch_matches_oracle(case):
    if case == "c1s":
        from cases import c1_problem
        bx, A = c1_problem(512, 8)
        tess = P.build_tessellation(P.grid_points(512, 1), 8)
        op, oop, gc = P.DenseOperator(A), O.Dense(A), 15
    elif case == "log1k":
        from cases import log_problem
        bx, coords, oop = log_problem(32, 16)
        tess = P.build_tessellation(P.grid_points(32, 2), 16)
        op, gc = P.KernelOperator(coords, "log", oop.diag), 15
    elif case == "inv1k":
        coords = O.cell_centres(32, 2)
        bx, oop = O.partition(coords, 16), O.KernelOp(coords, "inv", 64.0)
        tess = P.build_tessellation(P.grid_points(32, 2), 16)
        op, gc = P.KernelOperator(coords, "inv", 64.0), 15
    elif case == "inv3d":
        coords = O.cell_centres(12, 3)   # ell = 28: the general (v1) sketch
        bx, oop = O.partition(coords, 64), O.KernelOp(coords, "inv", 24.0)
        tess = P.build_tessellation(P.grid_points(12, 3), 64)
        op, gc = P.KernelOperator(coords, "inv", 24.0), 8
    else:
        from cases import rand500_problem
        bx, coords, oop = rand500_problem()
        tess = P.build_tessellation(P.PointCloud(coords, 2), 16)
        kind, diag = ("inv", 40.0) if case.startswith("inv") else ("log", 3.0)
        oop = O.KernelOp(coords, kind, diag)
        op, gc = P.KernelOperator(coords, kind, diag), 12
    dt = device_tess(tess, torch.device(DEV))
    st = P.RandomStream(7).child(0)
    plan = P.plan_tagging(tess, 0, "gaussian", P.RandomStream(7).child(1))
    G = draw_test_blocks(dt, st, 0, gc)
    H = draw_test_blocks(dt, st, 1, gc)
    T_dev = torch.from_numpy(plan.matrix.entries).to(DEV)
    Y, Z = tagged_sketch(op, dt, T_dev, plan.matrix.entries, G, H, gc)
    oplan = O.TagPlan(plan.matrix.entries, plan.Z, plan.rho_base, 1)
    _, bundle = O.bases_tagging(oop, bx, gc - 5 if gc > 5 else 1, 5, oplan, O.Stream(7).child(0), gc=gc)
    Yh, Zh = dt.from_perm_rows(Y), dt.from_perm_rows(Z)
    scale = np.linalg.norm(bundle.y)
    assert np.linalg.norm(Yh - bundle.y) <= 1e-13 * scale
    assert np.linalg.norm(Zh - bundle.z) <= 1e-13 * np.linalg.norm(bundle.z)
    # the compensated fold (type B): same products (ell > 10 falls back to the plain fold)
    Yc, Zc = tagged_sketch(op, dt, T_dev, plan.matrix.entries, G, H, gc, compensated=True)
    assert np.linalg.norm(dt.from_perm_rows(Yc) - bundle.y) <= 1e-13 * scale
    assert np.linalg.norm(dt.from_perm_rows(Zc) - bundle.z) <= 1e-13 * np.linalg.norm(bundle.z)


@pytest.mark.parametrize("kind,comp,rows,gc", [("log", 0, (0, 4096), 20), ("inv", 1, (512, 3100), 64),
                                                ("log", 1, (0, 4096), 30), ("inv", 0, (1000, 4096), 32)])
def test_tagged_sketch_staged_matches_fused(kind, comp, rows, gc):
    """ublr_sketch_tagged_staged (A evaluated once per strip of rows, copy-only
    producers) against the fused entry points on a row range, with a workspace
    of a few 32-row tiles (several strips, a ragged last one)."""
    per, nb = 64, 64
    coords = O.cell_centres(per, 2)
    n = len(coords)
    tess = P.build_tessellation(P.grid_points(per, 2), nb)
    op = P.KernelOperator(coords, kind, 4.0 if kind == "log" else 128.0)
    dt = device_tess(tess, torch.device(DEV))
    plan = P.plan_tagging(tess, 0, "gaussian", P.RandomStream(5).child(1))
    T = plan.matrix.entries
    ell = T.shape[1]
    st = P.RandomStream(5).child(0)
    G = draw_test_blocks(dt, st, 0, gc)
    H = draw_test_blocks(dt, st, 1, gc)
    T_dev = torch.from_numpy(T).to(DEV)
    s = ell * gc
    r0, r1 = rows
    outs = []
    for staged in (False, True):
        Y = torch.full((n, s), np.nan, dtype=torch.float64, device=DEV)
        Z = torch.full((n, s), np.nan, dtype=torch.float64, device=DEV)
        if staged:
            nbytes = 10 * 32 * n * 8            # ten row tiles per strip
            ws = torch.full((nbytes // 8,), np.nan, dtype=torch.float64, device=DEV)
            _lib.call("ublr_sketch_tagged_staged", op.device_op(dt.perm), _lib.ptr(dt.off), dt.b, _lib.ptr(T_dev), ell,
                      _lib.ptr(G), _lib.ptr(H), gc, gc, _lib.ptr(Y), _lib.ptr(Z), s, r0, r1, comp, _lib.ptr(ws),
                      nbytes, _lib.stream_handle())
        else:
            _lib.call("ublr_sketch_tagged_comp" if comp else "ublr_sketch_tagged_pair", op.device_op(dt.perm),
                      _lib.ptr(dt.off), dt.b, _lib.ptr(T_dev), ell, _lib.ptr(G), _lib.ptr(H), gc, gc, _lib.ptr(Y),
                      _lib.ptr(Z), s, r0, r1, _lib.stream_handle())
        outs.append((Y.cpu().numpy(), Z.cpu().numpy()))
    for a, b_ in zip(outs[0], outs[1]):
        assert np.isnan(a[:r0]).all() and np.isnan(a[r1:]).all() and np.isnan(b_[:r0]).all() and np.isnan(b_[r1:]).all()
        assert np.isfinite(b_[r0:r1]).all()
        assert np.linalg.norm(a[r0:r1] - b_[r0:r1]) <= 1e-14 * np.linalg.norm(a[r0:r1])


@pytest.mark.parametrize("kind", ["log", "dense"])
def test_tagged_sketch_compensated_fold_is_more_accurate(kind):
    """Against an 80-bit (numpy longdouble) evaluation of Y = A Omega on a
    64-block problem, the compensated fold's error is below the plain fold's
    (kernel operator: the warp-specialised kernel with bf16 error sums;
    dense A: the register-tile kernel)."""
    per, nb, gc = 64, 64, 20
    coords = O.cell_centres(per, 2)
    n = len(coords)
    tess = P.build_tessellation(P.grid_points(per, 2), nb)
    A = O.kernel_block(coords, np.arange(n), np.arange(n), "log", 4.0)
    op = P.KernelOperator(coords, "log", 4.0) if kind == "log" else P.DenseOperator(A)
    dt = device_tess(tess, torch.device(DEV))
    st = P.RandomStream(5).child(0)
    plan = P.plan_tagging(tess, 0, "gaussian", P.RandomStream(5).child(1))
    T = plan.matrix.entries
    G = draw_test_blocks(dt, st, 0, gc)
    H = draw_test_blocks(dt, st, 1, gc)
    T_dev = torch.from_numpy(T).to(DEV)
    Y0, _ = tagged_sketch(op, dt, T_dev, T, G, H, gc)
    Y1, _ = tagged_sketch(op, dt, T_dev, T, G, H, gc, compensated=True)
    # reference in extended precision, permuted row order; A as the device evaluates it
    Ad = op.apply(np.eye(n)) if kind == "log" else A
    Ap = Ad[np.ix_(dt.perm_h, dt.perm_h)].astype(np.longdouble)
    Gh = G.cpu().numpy().astype(np.longdouble)
    ref = np.zeros((n, T.shape[1] * gc), dtype=np.longdouble)
    for j in range(nb):
        r0, r1 = int(dt.off_h[j]), int(dt.off_h[j + 1])
        Wj = Ap[:, r0:r1] @ Gh[r0:r1]
        for c in range(T.shape[1]):
            ref[:, c * gc:(c + 1) * gc] += np.longdouble(T[j, c]) * Wj
    e0 = float(np.linalg.norm((Y0.cpu().numpy().astype(np.longdouble) - ref).astype(float)))
    e1 = float(np.linalg.norm((Y1.cpu().numpy().astype(np.longdouble) - ref).astype(float)))
    print(f"tagged sketch error vs 80-bit: plain {e0:.3e} compensated {e1:.3e}")
    assert e1 <= 0.9 * e0


@pytest.mark.parametrize("m,n,k", [(64, 20, 10), (256, 60, 48), (33, 33, 33), (100, 7, 7), (64, 40, 32), (17, 5, 5)])
def test_col_basis_matches_numpy(m, n, k):
    B = np.random.default_rng(m + n).standard_normal((m, n))
    got = P.col_basis(B, k)
    want = O.leading_q(B, k)
    assert np.abs(got - want).max() <= 1e-12


# ---------------------------------------------------------------- dense toolkit
from paper_2501_05528_b200 import dense as Dn  # noqa: E402


@pytest.mark.parametrize("n", [64, 150, 300])
def test_blocked_cholesky_and_trsm(n):
    rng = np.random.default_rng(n)
    batch = 3
    Bm = rng.standard_normal((batch, n, n + 20))
    Gh = Bm @ Bm.transpose(0, 2, 1)
    G = torch.from_numpy(Gh.copy()).cuda()
    R = torch.zeros_like(G)
    f = Dn.cholesky_upper(G, R)
    Dn.check_status(f, "chol")
    Rh = R.cpu().numpy()
    for b in range(batch):
        want = np.linalg.cholesky(Gh[b]).T
        assert np.abs(Rh[b] - want).max() <= 1e-10 * np.abs(want).max()
    X = torch.from_numpy(rng.standard_normal((batch, 37, n))).cuda()
    Xh = X.cpu().numpy()
    Dn.trsm_right_upper(X, R, f, torch.empty((batch, 37, Dn.NB), dtype=torch.float64, device="cuda"))
    for b in range(batch):
        assert np.abs(X.cpu().numpy()[b] @ Rh[b] - Xh[b]).max() <= 1e-11 * np.abs(Xh[b]).max()
    for upper, trans in ((True, True), (True, False)):
        Y = torch.from_numpy(rng.standard_normal((batch, n, 5))).cuda()
        Yh = Y.cpu().numpy()
        Dn.trsm_left(R, Y, f, f.inv, upper=upper, trans=trans,
                     tmp=torch.empty((batch, Dn.NB, 5), dtype=torch.float64, device="cuda"))
        for b in range(batch):
            T = Rh[b].T if trans else Rh[b]
            assert np.abs(T @ Y.cpu().numpy()[b] - Yh[b]).max() <= 1e-10 * np.abs(Yh[b]).max()


def test_lu_sign_reconstructs_householder():
    """LU of D - Qt_top with the sign rule gives LAPACK's tau in [1, 2]."""
    rng = np.random.default_rng(3)
    n, s = 130, 150
    B = rng.standard_normal((n, s))
    Qt = np.linalg.qr(B.T)[0]            # some thin Q (signs arbitrary)
    W = torch.from_numpy((-Qt[:n])[None].copy()).cuda()
    LU = torch.zeros_like(W)
    Dg = torch.zeros((1, n), dtype=torch.float64, device="cuda")
    f = Dn.lu_sign(W, LU, Dg)
    Dn.check_status(f, "lu")
    LUh, d = LU.cpu().numpy()[0], Dg.cpu().numpy()[0]
    L = np.tril(LUh, -1) + np.eye(n)
    U = np.triu(LUh)
    assert np.abs(L @ U - (np.diag(d) - Qt[:n])).max() <= 1e-12
    tau = np.diag(U) * d
    assert tau.min() >= 1.0 - 1e-12 and tau.max() <= 2.0 + 1e-12


def test_lu_sign_r_scaled_matches_unscaled_l():
    """LU of D R - B1^T (R = chol(B B^T)) has the L and signs of LU(D - Q_top)
    with Q_top = B1^T R^-1, and U' = U R (the bn null-space shortcut)."""
    rng = np.random.default_rng(5)
    n, s, batch = 200, 230, 3
    Bs = rng.standard_normal((batch, n, s))
    Rh = np.ascontiguousarray(np.stack([np.linalg.cholesky(b @ b.T).T for b in Bs]))
    B1T = np.ascontiguousarray(np.stack([b[:, :n].T for b in Bs]))
    W = torch.from_numpy(-B1T).cuda()
    R = torch.from_numpy(Rh).cuda()
    LU = torch.zeros_like(W)
    Dg = torch.zeros((batch, n), dtype=torch.float64, device="cuda")
    f = Dn.lu_sign(W, LU, Dg, R=R)
    Dn.check_status(f, "lu")
    W0 = torch.from_numpy(-np.ascontiguousarray(np.stack([np.linalg.solve(Rh[b].T, B1T[b].T).T
                                                          for b in range(batch)]))).cuda()
    LU0 = torch.zeros_like(W0)
    D0 = torch.zeros_like(Dg)
    Dn.check_status(Dn.lu_sign(W0, LU0, D0), "lu")
    assert torch.equal(Dg, D0)
    for b in range(batch):
        A, A0 = LU[b].cpu().numpy(), LU0[b].cpu().numpy()
        assert np.abs(np.tril(A, -1) - np.tril(A0, -1)).max() <= 1e-10
        assert np.abs(np.triu(A) - np.triu(A0) @ Rh[b]).max() <= 1e-10 * np.abs(np.triu(A)).max()


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K,batch", [(300, 200, 77, 3), (131, 45, 33, 2), (1000, 1100, 129, 1), (64, 40, 65, 5),
                                         (257, 300, 1, 2)])
@pytest.mark.parametrize("pad", [3, 4])
def test_gemm_batched_ragged_shapes(ta, tb, M, N, K, batch, pad):
    """Every orientation on shapes that end inside a tile in all three
    dimensions (the operand tiles are zero-filled only where the k dimension
    runs out; the rest of a ragged tile is left as it is), the operands
    embedded in NaN so that a read outside (M, N, K) shows."""
    rng = np.random.default_rng(M + N + K)   # pad 4: 16-byte-aligned operands (vector copies) when the ld is even

    def embed(x):
        out = np.full((x.shape[0], x.shape[1] + pad, x.shape[2] + 2 * pad), np.nan)
        out[:, :x.shape[1], pad:pad + x.shape[2]] = x
        return torch.from_numpy(out).cuda()

    A = rng.standard_normal((batch, K, M) if ta else (batch, M, K))
    B = rng.standard_normal((batch, N, K) if tb else (batch, K, N))
    C0 = rng.standard_normal((batch, M, N))
    Ad, Bd = embed(A), embed(B)
    Cd = torch.from_numpy(C0).cuda()
    want = 0.5 * C0 - np.einsum("bmk,bkn->bmn", A.transpose(0, 2, 1) if ta else A, B.transpose(0, 2, 1) if tb else B)
    Dn.gemm(ta, tb, M, N, K, -1.0, Dn.addr(Ad, pad), Ad.shape[2], Ad[0].numel(), Dn.addr(Bd, pad), Bd.shape[2],
            Bd[0].numel(), 0.5, Dn.addr(Cd), N, M * N, batch)
    got = Cd.cpu().numpy()
    assert np.isfinite(got).all()
    assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("kind,per,w", [("log", 70, 700), ("inv", 67, 1100), ("log", 64, 513)])
def test_apply_staged_matches_fused(kind, per, w):
    """ublr_apply_staged (A evaluated once per strip of rows, then the
    stored-operand GEMM) against ublr_apply (A evaluated inside the GEMM) and
    numpy, with a workspace of exactly two 128-row strips (several strips, a
    ragged last one) and with the library's own size."""
    coords = O.cell_centres(per, 2)
    n = len(coords)
    op = P.KernelOperator(coords, kind, 3.25)
    perm = torch.arange(n, dtype=torch.int32, device=DEV)
    X = torch.from_numpy(np.random.default_rng(4).standard_normal((n, w))).cuda()
    fused = torch.empty((n, w), dtype=torch.float64, device=DEV)
    _lib.call("ublr_apply", op.device_op(perm), X.data_ptr(), w, w, fused.data_ptr(), w, _lib.stream_handle())
    A = O.kernel_block(coords, np.arange(n), np.arange(n), kind, 3.25)
    want = A @ X.cpu().numpy()
    scale = np.linalg.norm(A) * np.linalg.norm(X.cpu().numpy())
    lib = _lib.load()
    for nbytes in (2 * 128 * n * 8, int(lib.ublr_apply_staged_workspace_bytes(n, w))):
        ws = torch.full((nbytes // 8,), np.nan, dtype=torch.float64, device=DEV)
        out = torch.full((n, w), np.nan, dtype=torch.float64, device=DEV)
        _lib.call("ublr_apply_staged", op.device_op(perm), X.data_ptr(), w, w, out.data_ptr(), w, ws.data_ptr(),
                  nbytes, _lib.stream_handle())
        got = out.cpu().numpy()
        assert np.linalg.norm(got - want) <= 1e-13 * scale
        assert np.linalg.norm(got - fused.cpu().numpy()) <= 1e-13 * scale
    with pytest.raises(ValueError):
        _lib.call("ublr_apply_staged", op.device_op(perm), X.data_ptr(), w, w, out.data_ptr(), w, ws.data_ptr(),
                  64 * n * 8, _lib.stream_handle())


def test_syrk_upper_matches_gemm_on_upper_triangle():
    rng = np.random.default_rng(6)
    for M, K in ((300, 64), (77, 13)):
        A = torch.from_numpy(rng.standard_normal((2, K, M))).cuda()
        C = torch.from_numpy(rng.standard_normal((2, M, M))).cuda()
        ref = C.cpu().numpy() - np.einsum("bki,bkj->bij", A.cpu().numpy(), A.cpu().numpy())
        _lib.call("ublr_syrk_upper_batched", M, K, -1.0, A.data_ptr(), M, K * M, 1.0, C.data_ptr(), M, M * M, 2,
                  _lib.stream_handle())
        iu = np.triu_indices(M)
        got = C.cpu().numpy()
        assert np.abs(got[:, iu[0], iu[1]] - ref[:, iu[0], iu[1]]).max() <= 1e-11


def test_nullspace_samples_match_reference_null_basis():
    from paper_2501_05528_b200.bases import nullspace_samples
    pts = P.grid_points(32, 2)
    tess = P.build_tessellation(pts, 16)
    dt = device_tess(tess, torch.device(DEV))
    k, p = 8, 4
    r = k + p
    s = P.block_nullification_width(tess, r)
    rng = np.random.default_rng(11)
    Om = rng.standard_normal((dt.n, s))          # original row order
    Yh = rng.standard_normal((dt.n, s))
    OP = dt.to_perm_rows(Om)
    Yd = dt.to_perm_rows(Yh)
    S = torch.zeros((dt.n, k), dtype=torch.float64, device=DEV)
    nullspace_samples(dt, OP, s, 0, Yd, s, s, r, k, S)
    Sh = dt.from_perm_rows(S)
    for i in range(tess.b):
        nbr = tess.neighbor_indices(i)
        Pk = O.null_tail(Om[nbr], r)[:, :k]
        want = Yh[tess.blocks[i]] @ Pk
        got = Sh[tess.blocks[i]]
        assert np.abs(got - want).max() <= 1e-11 * np.abs(want).max(), i


@pytest.mark.parametrize("per,b", [(32, 16), (48, 9)])
def test_nullspace_samples_both_sides_in_one_batch(per, b):
    """nside = 2 (both block-nullification sides in the same launches, virtual
    row maps into [Omega | Psi] and [Y | Z]) equals two one-side calls."""
    from paper_2501_05528_b200.bases import nullspace_samples
    tess = P.build_tessellation(P.grid_points(per, 2), b)
    dt = device_tess(tess, torch.device(DEV))
    k, p = 8, 4
    r = k + p
    s = P.block_nullification_width(tess, r)
    rng = np.random.default_rng(5)
    OP = torch.from_numpy(rng.standard_normal((dt.n, 2 * s))).to(DEV)
    YZ = torch.from_numpy(rng.standard_normal((dt.n, 2 * s))).to(DEV)
    both = torch.zeros((dt.n, 2, k), dtype=torch.float64, device=DEV)
    nullspace_samples(dt, OP, 2 * s, 0, YZ, 2 * s, s, r, k, both, nside=2)
    for side in (0, 1):
        one = torch.zeros((dt.n, k), dtype=torch.float64, device=DEV)
        nullspace_samples(dt, OP, 2 * s, side * s, YZ[:, side * s:], 2 * s, s, r, k, one)
        d = (both[:, side] - one).abs().max().item()
        assert d <= 1e-12 * one.abs().max().item(), (side, d)


@pytest.mark.parametrize("kind,k,per,nb", [("inv", 48, 64, 16), ("log", 40, 64, 16), ("log", 33, 50, 16)])
def test_coupling_matches_numpy(kind, k, per, nb):
    """C_ij = U_i^T A_ij V_j for every block pair (the m = 256 warp-specialised
    coupling, and ragged 256-point blocks for per = 48)."""
    from paper_2501_05528_b200.bases import BlockBases
    from paper_2501_05528_b200.reconstruction import direct_core
    pts = P.grid_points(per, 2)
    tess = P.build_tessellation(pts, nb)
    dt = device_tess(tess, torch.device(DEV))
    diag = -np.log(0.5 / per) if kind == "log" else 2.0 * per
    op = P.KernelOperator(pts, kind, diag)
    rng = np.random.default_rng(17)
    n = dt.n
    Uh, Vh = rng.standard_normal((n, k)), rng.standard_normal((n, k))
    bs = BlockBases(dt, torch.from_numpy(Uh).cuda(), torch.from_numpy(Vh).cuda(), k, "tag", (0, 0))
    core = direct_core(op, tess, bs).cpu().numpy()
    coords = pts.coords if hasattr(pts, "coords") else np.asarray(pts)
    perm = dt.perm_h if hasattr(dt, "perm_h") else None
    off = dt.off_h
    roff = dt.roff(k)[0]
    for i in range(dt.b):
        for j in range(dt.b):
            ri = perm[off[i]:off[i + 1]] if perm is not None else np.arange(off[i], off[i + 1])
            cj = perm[off[j]:off[j + 1]] if perm is not None else np.arange(off[j], off[j + 1])
            A = O.kernel_block(coords, ri, cj, kind, diag)
            ki, kj = roff[i + 1] - roff[i], roff[j + 1] - roff[j]
            ref = Uh[off[i]:off[i + 1], :ki].T @ A @ Vh[off[j]:off[j + 1], :kj]
            got = core[roff[i]:roff[i + 1], roff[j]:roff[j + 1]]
            assert np.abs(got - ref).max() <= 1e-11 * max(1.0, np.abs(ref).max()), (i, j)


@pytest.mark.parametrize("per,nb,d", [(64, 64, 2), (256, 1024, 2), (16, 64, 3)])
def test_tag_aspect_device_matches_host(per, nb, d):
    """GPU aspect ratios (ublr_tag_aspect) against the host |T Z^T| form, and
    the same redraw decisions for the whole policy."""
    from paper_2501_05528_b200.tagging import _evaluate, make_tagging_matrix
    tess = P.build_tessellation(P.grid_points(per, d), nb)
    T = make_tagging_matrix(tess.b, d, 0, "gaussian", P.RandomStream(3).child(1).child(0))
    h = _evaluate(T, tess, 1, device=False).rho_base
    g = _evaluate(T, tess, 1, device=True).rho_base
    assert np.array_equal(np.isnan(h), np.isnan(g))
    fin = np.isfinite(h)
    assert np.array_equal(fin, np.isfinite(g))
    # fma (device) vs separate multiply-add (host) dot products: rho = hi/lo
    # amplifies the rounding of a small lo
    assert np.allclose(g[fin], h[fin], rtol=1e-8, atol=0)
    ph = P.plan_tagging(tess, 0, "gaussian", P.RandomStream(3).child(1))
    pg = P.plan_tagging(tess, 0, "gaussian", P.RandomStream(3).child(1), device=True)
    assert ph.attempts == pg.attempts and np.array_equal(ph.matrix.entries, pg.matrix.entries)


def _fused_case(name):
    if name == "dense1d":
        pts = P.grid_points(512, 1)
        tess = P.build_tessellation(pts, 8)
        A = np.random.default_rng(3).standard_normal((512, 512))
        return tess, P.DenseOperator(A)
    if name == "log2d":
        pts = P.grid_points(32, 2)
        return P.build_tessellation(pts, 16), P.KernelOperator(pts, "log", -np.log(0.5 / 32))
    if name == "inv_ragged":
        pts = P.grid_points(48, 2)   # 36-point blocks
        return P.build_tessellation(pts, 64), P.KernelOperator(pts, "inv", 96.0)
    if name == "log_rand":
        pts = P.random_points(500, 2, P.RandomStream(21))
        return P.build_tessellation(pts, 16), P.KernelOperator(pts, "log", 3.0)
    raise KeyError(name)


@pytest.mark.parametrize("name,k", [("dense1d", 10), ("log2d", 20), ("inv_ragged", 32), ("log_rand", 20),
                                    ("log2d", 7), ("log_rand", 30)])
def test_coupling_nearfield_fused_matches_separate(name, k):
    """ublr_coupling_nearfield (one pass over A for m <= 64) against the
    separate coupling + colour-probe kernels on the same U, V."""
    from paper_2501_05528_b200.bases import BlockBases
    from paper_2501_05528_b200.reconstruction import direct_core, structured_identity_discrepancy
    from paper_2501_05528_b200.tessellation import color_boxes
    tess, op = _fused_case(name)
    dt = device_tess(tess, torch.device(DEV))
    assert dt.m_max <= 64 and dt.pair_of is not None
    rng = np.random.default_rng(5)
    U = torch.from_numpy(rng.standard_normal((dt.n, k))).cuda()
    V = torch.from_numpy(rng.standard_normal((dt.n, k))).cuda()
    bs = BlockBases(dt, U, V, k, "tag", (0, 0))
    core_f = direct_core(op, tess, bs)
    assert getattr(bs, "fused_near", None) is not None
    B_f = structured_identity_discrepancy(op, tess, bs, core_f, color_boxes(tess)).cpu().numpy()
    # separate kernels
    K = bs.total_rank
    roff = dt.roff(k)[1]
    core_s = torch.empty_like(core_f)
    _lib.call("ublr_coupling", op.device_op(dt.perm), _lib.ptr(dt.off), _lib.ptr(roff), dt.b, k, _lib.ptr(U),
              _lib.ptr(V), k, _lib.ptr(core_s), K, _lib.stream_handle(), dt.m_max, 0, dt.b)
    bs.fused_near = None
    B_s = structured_identity_discrepancy(op, tess, bs, core_s, color_boxes(tess)).cpu().numpy()
    cf, cs = core_f.cpu().numpy(), core_s.cpu().numpy()
    assert np.abs(cf - cs).max() <= 1e-12 * np.abs(cs).max()
    assert B_f.shape == B_s.shape
    assert np.abs(B_f - B_s).max() <= 1e-12 * np.abs(B_s).max()
    # a modified core is not served from the fused pass
    direct_core(op, tess, bs)
    core2 = direct_core(op, tess, bs)
    core2.mul_(2.0)
    assert structured_identity_discrepancy(op, tess, bs, core2, color_boxes(tess)) is not bs.fused_near[3]


@pytest.mark.parametrize("per,nb,d,extra", [(64, 64, 2, 0), (32, 16, 2, 0), (12, 64, 3, 0), (64, 64, 2, 3),
                                           (64, 256, 2, 0)])
def test_null_vectors_device_bitwise_equal_host(per, nb, d, extra):
    """ublr_null_vectors_device gives the host planner's null vectors and
    residuals bit for bit (the pipeline's speculative block QR relies on it)."""
    from paper_2501_05528_b200.tagging import _neighbour_csr, make_tagging_matrix
    tess = P.build_tessellation(P.grid_points(per, d), nb)
    T = make_tagging_matrix(tess.b, d, extra, "gaussian", P.RandomStream(3).child(1).child(0))
    E = np.ascontiguousarray(T.entries)
    b, ell = E.shape
    ptr, idx = _neighbour_csr(tess)
    Zh, rh = np.zeros((b, ell)), np.zeros(b)
    _lib.check(_lib.load().ublr_null_vectors(E.ctypes.data, ell, ptr.ctypes.data, idx.ctypes.data, b,
                                             Zh.ctypes.data, rh.ctypes.data))
    dt = device_tess(tess, torch.device(DEV))
    Ed = torch.from_numpy(E).to(DEV)
    Zd = torch.empty((b, ell), dtype=torch.float64, device=DEV)
    rd = torch.empty(b, dtype=torch.float64, device=DEV)
    _lib.call("ublr_null_vectors_device", _lib.ptr(Ed), ell, _lib.ptr(dt.nptr), _lib.ptr(dt.nidx), b, _lib.ptr(Zd),
              _lib.ptr(rd), _lib.stream_handle())
    assert np.array_equal(Zd.cpu().numpy(), Zh)
    assert np.array_equal(rd.cpu().numpy(), rh)
