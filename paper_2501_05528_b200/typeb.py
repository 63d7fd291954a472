"""Type-B reconstruction on the GPU (ref/reconstruction.py:252-421).

* `tagging_pinv_discrepancy` (B2): near blocks from the wide tagging sketches
  with per-pair null vectors and the right pseudo-inverses of the test blocks.
* `gaussian_pinv_discrepancy` (B1): near blocks from the block-nullification
  sketches with the right pseudo-inverse of Omega[nbr(i)].
* `pinv_core`: C = U^T (Y - B Omega) (V^T Omega)^+ with Gaussian augmentation.

Right pseudo-inverses of full-row-rank matrices are formed through Cholesky
factorisations of Gram matrices (CholeskyQR2 for the K x (K+p) core system);
the reference uses SVDs with 1e-12 truncation, which never truncates for
these well-conditioned Gaussian test matrices (DESIGN.md §type B). A
rank-deficient system raises numpy.linalg.LinAlgError instead of truncating.
"""

from __future__ import annotations

import warnings

import numpy as np

from . import _lib
from . import dense as D
from .linalg import device_normals
from .operators import CountingOperator, unwrap
from .tagging import DegenerateTagsError, pair_vectors


def _torch():
    import torch
    return torch


def _f64(dev):
    import torch
    return dict(dtype=torch.float64, device=dev)


def _uniform(dt, what):
    if not (dt.sizes == dt.sizes[0]).all():
        raise NotImplementedError(f"{what}: the GPU path needs equal block sizes")
    return int(dt.sizes[0])


def _row_maps(dt, blocks, m):
    """(len(blocks), m) int32 device map of the permuted rows of each block."""
    torch = _torch()
    rows = dt.off_h[np.asarray(blocks)][:, None] + np.arange(m)[None, :]
    return torch.from_numpy(rows.astype(np.int32)).to(dt.device)


def right_pinv_T(dt, Gm):
    """pinv(G_j)^T = (G_j G_j^T)^-1 G_j for every block (G: N x gc, permuted
    rows), returned as an N x gc tensor; ref/linalg.py:97-109 applied per block
    at ref/reconstruction.py:341-342."""
    torch = _torch()
    m = _uniform(dt, "right_pinv_T")
    b, gc = dt.b, Gm.shape[1]
    Gr = torch.empty((b, m, m), **_f64(dt.device))
    R = torch.zeros_like(Gr)
    D.gemm(0, 1, m, m, gc, 1.0, D.addr(Gm), gc, m * gc, D.addr(Gm), gc, m * gc, 0.0, D.addr(Gr), m, m * m, b)
    f = D.cholesky_upper(Gr, R)
    X = Gm.clone().reshape(b, m, gc)
    tmp = torch.empty((b, D.NB, gc), **_f64(dt.device))
    D.trsm_left(R, X, f, f.inv, upper=True, trans=True, tmp=tmp)
    D.trsm_left(R, X, f, f.inv, upper=True, trans=False, tmp=tmp)
    D.check_status(f, "pinv of a test block")
    return X.reshape(dt.n, gc)


def _perp_pairs(dt, Ub, ldu, k, comb, width, blocks_of_pairs, m):
    """comb_p <- comb_p - U_i (U_i^T comb_p), i = blocks_of_pairs[p] (in place)."""
    torch = _torch()
    P = comb.shape[0]
    amap = _row_maps(dt, blocks_of_pairs, m)
    T1 = torch.empty((P, k, width), **_f64(dt.device))
    D.gemm(1, 0, k, width, m, 1.0, D.addr(Ub), ldu, 0, D.addr(comb), width, m * width, 0.0, D.addr(T1), width,
           k * width, P, amap=D.addr(amap), sAm=m)
    D.gemm(0, 0, m, width, k, -1.0, D.addr(Ub), ldu, 0, D.addr(T1), width, k * width, 1.0, D.addr(comb), width,
           m * width, P, amap=D.addr(amap), sAm=m)
    return amap


def assemble_near(dt, left, Xadj, U, k, m):
    """B_p = left_p + U_i (U_i^T W_ij) with W_ij = Xadj_{tp}^T, tp the pair (j, i)
    (the recombination of ref/reconstruction.py:305 / :375, sign '+').
    left: (P, m, m) becomes B."""
    torch = _torch()
    P = dt.n_pairs
    amap = _row_maps(dt, dt.pair_i_h, m)
    tmap = torch.from_numpy((dt.tpair_h[:, None].astype(np.int64) * m + np.arange(m)[None, :]).astype(np.int32)).to(dt.device)
    T2 = torch.empty((P, k, m), **_f64(dt.device))
    # T2_p = U_i^T Xadj_tp^T
    D.gemm(1, 1, k, m, m, 1.0, D.addr(U), U.stride(0), 0, D.addr(Xadj), m, 0, 0.0, D.addr(T2), m, k * m, P,
           amap=D.addr(amap), sAm=m, bmap=D.addr(tmap), sBm=m)
    D.gemm(0, 0, m, m, k, 1.0, D.addr(U), U.stride(0), 0, D.addr(T2), m, k * m, 1.0, D.addr(left), m, m * m, P,
           amap=D.addr(amap), sAm=m)
    return left.reshape(-1)


def tagging_pinv_discrepancy(bundle, bases, denom_rtol: float = 1e-10):
    """B2 near blocks (ref/reconstruction.py:326-376). Returns the flat device
    buffer of near blocks in neighbour-CSR order."""
    torch = _torch()
    dt = bases.dt
    m = _uniform(dt, "tagging_pinv_discrepancy")
    k = int(min(bases.rank, m))
    T = bundle.tagging.entries
    ell = T.shape[1]
    gc = bundle.group_cols
    Zp, den = pair_vectors(T, dt.tess, denom_rtol)
    w = torch.from_numpy(np.ascontiguousarray(Zp / den[:, None])).to(dt.device)
    GpT = right_pinv_T(dt, bundle.G)
    HpT = right_pinv_T(dt, bundle.H)
    P = dt.n_pairs
    st = _lib.stream_handle()
    f64 = _f64(dt.device)
    out = []
    for Ysrc, Ub, PinvT in ((bundle.Y, bases.U, GpT), (bundle.Z, bases.V, HpT)):
        comb = torch.empty((P, m, gc), **f64)
        _lib.call("ublr_tag_combine_pairs", D.addr(Ysrc), Ysrc.stride(0), gc, ell, D.addr(w), D.addr(dt.pair_i),
                  D.addr(dt.off), P, m, D.addr(comb), st)
        _perp_pairs(dt, Ub, Ub.stride(0), k, comb, gc, dt.pair_i_h, m)
        # X_p = comb_p pinv(G_other)   (other = nidx[p]); pinv(G)^T rows gathered by bmap
        bmap = _row_maps(dt, dt.nidx_h, m)
        X = torch.empty((P, m, m), **f64)
        D.gemm(0, 1, m, m, gc, 1.0, D.addr(comb), gc, m * gc, D.addr(PinvT), gc, 0, 0.0, D.addr(X), m, m * m, P,
               bmap=D.addr(bmap), sBm=m)
        out.append(X)
    return assemble_near(dt, out[0], out[1], bases.U, k, m)


def _gram_chol(dt, Om, ld_om, amap, n, s, nb_):
    torch = _torch()
    f64 = _f64(dt.device)
    G = torch.empty((nb_, n, n), **f64)
    R = torch.zeros_like(G)
    D.gemm(0, 1, n, n, s, 1.0, D.addr(Om), ld_om, 0, D.addr(Om), ld_om, 0, 0.0, D.addr(G), n, n * n, nb_,
           amap=D.addr(amap), sAm=n, bmap=D.addr(amap), sBm=n)
    f = D.cholesky_upper(G, R)
    return R, f


def _cond_estimate(R):
    """Lower bound of cond(Omega[nbr]) = cond(R): max|R_jj| / min|R_jj| (the
    reference's exact s_max/s_min comes from an SVD; DESIGN.md §type B)."""
    d = R.diagonal(dim1=1, dim2=2).abs()
    return (d.max(dim=1).values / d.min(dim=1).values).cpu().numpy()


def gaussian_pinv_discrepancy(bundle, bases, cond_limit: float = 1e8):
    """B1 near blocks (ref/reconstruction.py:266-307)."""
    torch = _torch()
    dt = bases.dt
    m = _uniform(dt, "gaussian_pinv_discrepancy")
    k = int(min(bases.rank, m))
    s = bundle.s
    P = dt.n_pairs
    f64 = _f64(dt.device)
    sizes = dt.sizes
    nbr_n = np.array([int(sizes[dt.nidx_h[dt.nptr_h[i]:dt.nptr_h[i + 1]]].sum()) for i in range(dt.b)])
    side_out = []
    for Om_d, Ysrc, Ub, label in ((bundle._omega_d, bundle.Y, bases.U, "neighbor"),
                                  (bundle._psi_d, bundle.Z, bases.V, "neighbor adjoint")):
        pieces = torch.empty((P, m, m), **f64)      # per pair (i, j): x_i[:, cols of j]
        for n in np.unique(nbr_n):
            n = int(n)
            blk = np.flatnonzero(nbr_n == n)
            nb_ = len(blk)
            maps = np.stack([np.concatenate([np.arange(dt.off_h[j], dt.off_h[j + 1])
                                             for j in dt.nidx_h[dt.nptr_h[i]:dt.nptr_h[i + 1]]]) for i in blk])
            amap = torch.from_numpy(maps.astype(np.int32)).to(dt.device)
            R, f = _gram_chol(dt, Om_d, Om_d.stride(0), amap, n, s, nb_)
            D.check_status(f, "Gram of Omega[nbr]")
            cond = _cond_estimate(R)
            for bi, c in zip(blk, cond):
                if c > cond_limit:
                    warnings.warn(f"block {bi}: {label} test-matrix stack has condition {c:.2e}")
            rmap = _row_maps(dt, blk, m)
            # Py = Y_i - U_i (U_i^T Y_i)   (m x s)
            Py = torch.empty((nb_, m, s), **f64)
            _lib.call("ublr_gather", D.addr(Ysrc), Ysrc.stride(0), 0, D.addr(rmap), m, m, s, 0, 0, D.addr(Py), s,
                      m * s, nb_, _lib.stream_handle())
            _perp_pairs(dt, Ub, Ub.stride(0), k, Py, s, blk, m)
            # x = Py B^T G^-1 = ((Py B^T) R^-1) R^-T
            X = torch.empty((nb_, m, n), **f64)
            D.gemm(0, 1, m, n, s, 1.0, D.addr(Py), s, m * s, D.addr(Om_d), Om_d.stride(0), 0, 0.0, D.addr(X), n,
                   m * n, nb_, bmap=D.addr(amap), sBm=n)
            D.trsm_right_upper(X, R, f, torch.empty((nb_, m, D.NB), **f64))
            Xt = torch.empty((nb_, n, m), **f64)
            _lib.call("ublr_gather", D.addr(X), n, m * n, None, 0, m, n, 0, 1, D.addr(Xt), m, n * m, nb_,
                      _lib.stream_handle())
            D.trsm_left(R, Xt, f, f.inv, upper=True, trans=False, tmp=torch.empty((nb_, D.NB, m), **f64))
            # split x_i^T (n x m) by neighbour: pair p = nptr[i] + t holds rows t*m .. of x_i^T, transposed
            for li, i in enumerate(blk):
                for t in range(dt.nptr_h[i + 1] - dt.nptr_h[i]):
                    p = int(dt.nptr_h[i] + t)
                    _lib.call("ublr_gather", D.addr(Xt, li * n * m + t * m * m), m, 0, None, 0, m, m, 0, 1,
                              D.addr(pieces, p * m * m), m, 0, 1, _lib.stream_handle())
        side_out.append(pieces)
    return assemble_near(dt, side_out[0], side_out[1], bases.U, k, m)


def pinv_core(op, bundle, bases, B_flat, p: int, stream, max_width=None):
    """C = U^T (Y - B Omega) (V^T Omega)^+ (ref/reconstruction.py:379-421).
    Returns (core K x K device tensor, columns added)."""
    torch = _torch()
    dt = bases.dt
    m = _uniform(dt, "pinv_core")
    k = int(min(bases.rank, m))
    K = bases.total_rank
    s = bundle.s
    n = dt.n
    f64 = _f64(dt.device)
    extra = max(0, K + p - s)
    if extra and max_width is not None and s + extra > max_width:
        raise ValueError(f"type B needs sketch width {K + p} > max_width {max_width}")
    L = s + extra
    Of = torch.empty((n, L), **f64)
    Yf = torch.empty((n, L), **f64)
    st = _lib.stream_handle()
    if bundle.kind == "tag":
        _lib.call("ublr_assemble_tagged", D.addr(torch.from_numpy(np.ascontiguousarray(bundle.tagging.entries)).to(dt.device)),
                  bundle.tagging.entries.shape[1], D.addr(bundle.G), bundle.G.stride(0), bundle.group_cols,
                  D.addr(dt.off), dt.b, D.addr(Of), L, n, st)
    else:
        Of[:, :s].copy_(bundle._omega_d)
    Yf[:, :s].copy_(bundle.Y)
    if extra:
        device_normals([(stream, n, extra, s, L, dt.inv)], Of)
        if isinstance(op, CountingOperator):
            op.ledger.record_apply(extra)
        inner = unwrap(op)
        if hasattr(inner, "device_op"):
            _lib.call("ublr_apply", inner.device_op(dt.perm), D.addr(Of, s), L, extra, D.addr(Yf, s), L, st)
        else:
            Yf[:, s:] = dt.to_perm_rows(inner.apply(dt.from_perm_rows(Of[:, s:])))
    # Rf = Y - B Omega, accumulated by neighbour slot (no two writers per row block)
    Bm = B_flat.reshape(-1, m)
    maxn = int(np.max(np.diff(dt.nptr_h)))
    for t in range(maxn):
        blk = np.flatnonzero(np.diff(dt.nptr_h) > t)
        pairs = dt.nptr_h[blk] + t
        amap = torch.from_numpy((pairs[:, None].astype(np.int64) * m + np.arange(m)[None, :]).astype(np.int32)).to(dt.device)
        bmap = _row_maps(dt, dt.nidx_h[pairs], m)
        cmap = _row_maps(dt, blk, m)
        D.gemm(0, 0, m, L, m, -1.0, D.addr(Bm), m, 0, D.addr(Of), L, 0, 1.0, D.addr(Yf), L, 0, len(blk),
               amap=D.addr(amap), sAm=m, bmap=D.addr(bmap), sBm=m, cmap=D.addr(cmap), sCm=m)
    # Vt Omega and U^T (Y - B Omega): K x L, block rows of k
    rmap = _row_maps(dt, np.arange(dt.b), m)
    VtO = torch.empty((K, L), **f64)
    LHS = torch.empty((K, L), **f64)
    D.gemm(1, 0, k, L, m, 1.0, D.addr(bases.V), bases.V.stride(0), 0, D.addr(Of), L, 0, 0.0, D.addr(VtO), L, k * L,
           dt.b, amap=D.addr(rmap), sAm=m, bmap=D.addr(rmap), sBm=m)
    D.gemm(1, 0, k, L, m, 1.0, D.addr(bases.U), bases.U.stride(0), 0, D.addr(Yf), L, 0, 0.0, D.addr(LHS), L, k * L,
           dt.b, amap=D.addr(rmap), sAm=m, bmap=D.addr(rmap), sBm=m)
    del Of, Yf
    core = lstsq_right(LHS, VtO)
    return core, extra


def lstsq_right(LHS, M):
    """LHS M^+ for a full-row-rank M (K x L) by CholeskyQR2 of M^T:
    M^T = Q1 R1, Q1^T Q1 = R2^T R2, so M^+ = Q1 R2^-1 R2^-T R1^-T and
    (LHS M^+)^T = R1^-1 R2^-1 R2^-T (LHS Q1)^T."""
    torch = _torch()
    K, L = M.shape
    f64 = _f64(M.device)
    # Gram matrices by SYRK on M^T (upper tiles only: the Cholesky reads the upper triangle)
    Q1 = torch.empty((1, L, K), **f64)
    _lib.call("ublr_gather", D.addr(M), L, 0, None, 0, K, L, 0, 1, D.addr(Q1), K, 0, 1, _lib.stream_handle())
    G1 = torch.empty((1, K, K), **f64)
    R1 = torch.zeros_like(G1)
    D._syrk_upper(K, L, 1.0, D.addr(Q1), K, 0, 0.0, D.addr(G1), K, 0, 1)
    f1 = D.cholesky_upper(G1, R1)
    D.check_status(f1, "pinv_core: V^T Omega is rank deficient")
    D.trsm_right_upper(Q1, R1, f1, torch.empty((1, L, D.NB), **f64))
    G2 = torch.empty((1, K, K), **f64)
    R2 = torch.zeros_like(G2)
    D._syrk_upper(K, L, 1.0, D.addr(Q1), K, 0, 0.0, D.addr(G2), K, 0, 1)
    f2 = D.cholesky_upper(G2, R2)
    D.check_status(f2, "pinv_core: second CholeskyQR pass")
    C1t = torch.empty((1, K, LHS.shape[0]), **f64)      # (LHS Q1)^T = Q1^T LHS^T
    D.gemm(1, 1, K, LHS.shape[0], L, 1.0, D.addr(Q1), K, 0, D.addr(LHS), L, 0, 0.0, D.addr(C1t), LHS.shape[0], 0, 1)
    tmp = torch.empty((1, D.NB, LHS.shape[0]), **f64)
    D.trsm_left(R2, C1t, f2, f2.inv, upper=True, trans=True, tmp=tmp)
    D.trsm_left(R2, C1t, f2, f2.inv, upper=True, trans=False, tmp=tmp)
    D.trsm_left(R1, C1t, f1, f1.inv, upper=True, trans=False, tmp=tmp)
    core = torch.empty((LHS.shape[0], K), **f64)
    _lib.call("ublr_gather", D.addr(C1t), LHS.shape[0], 0, None, 0, K, LHS.shape[0], 0, 1, D.addr(core), K, 0, 1,
              _lib.stream_handle())
    return core
