"""Type-B reconstruction on the GPU (ref/reconstruction.py:252-421).

* `tagging_pinv_discrepancy` (B2): near blocks from the wide tagging sketches
  with per-pair null vectors and the right pseudo-inverses of the test blocks.
* `gaussian_pinv_discrepancy` (B1): near blocks from the block-nullification
  sketches with the right pseudo-inverse of Omega[nbr(i)].
* `pinv_core`: C = U^T (Y - B Omega) (V^T Omega)^+ with Gaussian augmentation.

Right pseudo-inverses of full-row-rank matrices are formed by CholeskyQR2
(per test block G_j, and for the K x (K+p) core system);
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
from .operators import CountingOperator, device_apply, unwrap
from .tagging import DegenerateTagsError, pair_vectors


def _torch():
    import torch
    return torch


def _f64(dev):
    import torch
    return dict(dtype=torch.float64, device=dev)


def _row_maps(dt, blocks, m):
    """(len(blocks), m) int32 device map of the permuted rows of each block."""
    torch = _torch()
    rows = dt.off_h[np.asarray(blocks)][:, None] + np.arange(m)[None, :]
    return torch.from_numpy(rows.astype(np.int32)).to(dt.device)


def _imap(dt, starts, width):
    """(len(starts), width) int32 device map starts[e] + 0 .. width-1."""
    torch = _torch()
    rows = np.asarray(starts, dtype=np.int64)[:, None] + np.arange(width)[None, :]
    return torch.from_numpy(rows.astype(np.int32)).to(dt.device)


def _size_groups(dt):
    """{m: blocks with m_i = m} (one entry on a uniform tessellation)."""
    out = {}
    for i, m in enumerate(dt.sizes.tolist()):
        out.setdefault(int(m), []).append(i)
    return {m: np.asarray(b) for m, b in sorted(out.items())}


def _pair_groups(dt, key):
    """Pairs p grouped by key(i, j) (i = pair_i[p], j = nidx[p])."""
    out = {}
    for p, (i, j) in enumerate(zip(dt.pair_i_h.tolist(), dt.nidx_h.tolist())):
        out.setdefault(key(i, j), []).append(p)
    return [(kk, np.asarray(v)) for kk, v in sorted(out.items())]


def right_pinv_T(dt, Gm):
    """pinv(G_j)^T for every block (G_j: m_j x gc rows of G, full row rank),
    returned as an N x gc tensor in G's layout; ref/linalg.py:97-109 applied
    per block at ref/reconstruction.py:341-342.

    CholeskyQR2 of G_j^T = Q R (R = R2 R1, G_j G_j^T = R1^T R1, Q1 = G_j^T R1^-1,
    Q1^T Q1 = R2^T R2): pinv(G_j)^T = R^-1 Q^T = R1^-1 R2^-1 R2^-T R1^-T G_j.
    The second pass removes the cond(G_j)^2 growth of the plain normal
    equations. Blocks are batched by size (ragged tessellations)."""
    torch = _torch()
    gc = Gm.shape[1]
    out = torch.empty_like(Gm)
    st = _lib.stream_handle()
    for m, bl in _size_groups(dt).items():
        nb = len(bl)
        rmap = _row_maps(dt, bl, m)
        X = torch.empty((nb, m, gc), **_f64(dt.device))
        _lib.call("ublr_gather", D.addr(Gm), gc, 0, D.addr(rmap), m, m, gc, 0, 0, D.addr(X), gc, m * gc, nb, st)
        tmp = torch.empty((nb, D.NB, gc), **_f64(dt.device))
        facs = []
        for _ in range(2):
            Gr = torch.empty((nb, m, m), **_f64(dt.device))
            R = torch.zeros_like(Gr)
            D.gemm(0, 1, m, m, gc, 1.0, D.addr(X), gc, m * gc, D.addr(X), gc, m * gc, 0.0, D.addr(Gr), m, m * m, nb)
            f = D.cholesky_upper(Gr, R)
            D.trsm_left(R, X, f, f.inv, upper=True, trans=True, tmp=tmp)      # X <- R^-T X
            facs.append((R, f))
        (R1, f1), (R2, f2) = facs
        D.trsm_left(R2, X, f2, f2.inv, upper=True, trans=False, tmp=tmp)      # R2^-1
        D.trsm_left(R1, X, f1, f1.inv, upper=True, trans=False, tmp=tmp)      # R1^-1
        D.check_status(f1, "pinv of a test block")
        D.check_status(f2, "pinv of a test block (second CholeskyQR pass)")
        if nb == dt.b:             # one size: the blocks tile the rows in order
            return X.view(dt.n, gc)
        out.index_copy_(0, rmap.reshape(-1).long(), X.view(nb * m, gc))
    return out


def _perp_rows(dt, Ub, k, buf, width, ld_rows, blocks_of, slots):
    """buf_s <- buf_s - U_i (U_i^T buf_s) for every slot s (rows slot*ld_rows + r
    of `buf`, width columns, ld = width), i = blocks_of[s]; batched per
    (m_i, k_i)."""
    torch = _torch()
    ranks = dt.ranks(k)
    groups = {}
    for s_, i in zip(slots, blocks_of):
        groups.setdefault((int(dt.sizes[i]), int(ranks[i])), []).append((s_, i))
    for (m, ki), mem in sorted(groups.items()):
        if ki == 0:
            continue
        sl = np.array([x[0] for x in mem])
        bl = np.array([x[1] for x in mem])
        umap = _row_maps(dt, bl, m)
        xmap = _imap(dt, sl * ld_rows, m)
        T1 = torch.empty((len(mem), ki, width), **_f64(dt.device))
        D.gemm(1, 0, ki, width, m, 1.0, D.addr(Ub), Ub.stride(0), 0, D.addr(buf), width, 0, 0.0, D.addr(T1), width,
               ki * width, len(mem), amap=D.addr(umap), sAm=m, bmap=D.addr(xmap), sBm=m)
        D.gemm(0, 0, m, width, ki, -1.0, D.addr(Ub), Ub.stride(0), 0, D.addr(T1), width, ki * width, 1.0,
               D.addr(buf), width, 0, len(mem), amap=D.addr(umap), sAm=m, cmap=D.addr(xmap), sCm=m)


def _pack(dt, padded):
    """Padded per-pair near blocks (P, m_max, m_max) -> flat neighbour-CSR
    buffer (views the padded buffer when every block has m_max points)."""
    torch = _torch()
    if (dt.sizes == dt.m_max).all():
        return padded.reshape(-1)
    flat = torch.empty(int(dt.b_off_h[-1]), **_f64(dt.device))
    _lib.call("ublr_pairs_pad", D.addr(flat), D.addr(dt.b_off), D.addr(dt.pair_i), D.addr(dt.nidx), D.addr(dt.off),
              dt.n_pairs, dt.m_max, D.addr(padded), 0, _lib.stream_handle())
    return flat


def assemble_near(dt, left, Xadj, U, k):
    """B_p = left_p + U_i (U_i^T W_ij) with W_ij = Xadj_{tp}^T, tp the pair (j, i)
    (the recombination of ref/reconstruction.py:305 / :375, sign '+').
    left, Xadj: padded (P, m_max, m_max); returns the flat near-block buffer."""
    torch = _torch()
    mm = dt.m_max
    ranks = dt.ranks(k)
    for (mi, mj, ki), ps in _pair_groups(dt, lambda i, j: (int(dt.sizes[i]), int(dt.sizes[j]), int(ranks[i]))):
        if ki == 0:
            continue
        np_ = len(ps)
        umap = _row_maps(dt, dt.pair_i_h[ps], mi)
        tmap = _imap(dt, dt.tpair_h[ps].astype(np.int64) * mm, mj)     # rows of X_tp (m_j x m_i)
        T2 = torch.empty((np_, ki, mj), **_f64(dt.device))
        D.gemm(1, 1, ki, mj, mi, 1.0, D.addr(U), U.stride(0), 0, D.addr(Xadj), mm, 0, 0.0, D.addr(T2), mj, ki * mj,
               np_, amap=D.addr(umap), sAm=mi, bmap=D.addr(tmap), sBm=mj)
        D.gemm(0, 0, mi, mj, ki, 1.0, D.addr(U), U.stride(0), 0, D.addr(T2), mj, ki * mj, 1.0, D.addr(left), mm, 0,
               np_, amap=D.addr(umap), sAm=mi, cmap=D.addr(_imap(dt, ps.astype(np.int64) * mm, mi)), sCm=mi)
    return _pack(dt, left)


def tagging_pinv_discrepancy(bundle, bases, denom_rtol: float = 1e-10):
    """B2 near blocks (ref/reconstruction.py:326-376). Returns the flat device
    buffer of near blocks in neighbour-CSR order (ragged blocks supported)."""
    torch = _torch()
    dt = bases.dt
    mm = dt.m_max
    k = bases.rank
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
        comb = torch.empty((P, mm, gc), **f64)
        _lib.call("ublr_tag_combine_pairs", D.addr(Ysrc), Ysrc.stride(0), gc, ell, D.addr(w), D.addr(dt.pair_i),
                  D.addr(dt.off), P, mm, D.addr(comb), st)
        _perp_rows(dt, Ub, k, comb, gc, mm, dt.pair_i_h, np.arange(P))
        # X_p = comb_p pinv(G_j)   (j = nidx[p]); pinv(G)^T rows gathered by bmap
        X = torch.empty((P, mm, mm), **f64)
        for (mi, mj), ps in _pair_groups(dt, lambda i, j: (int(dt.sizes[i]), int(dt.sizes[j]))):
            rmap = _imap(dt, ps.astype(np.int64) * mm, mi)
            D.gemm(0, 1, mi, mj, gc, 1.0, D.addr(comb), gc, 0, D.addr(PinvT), gc, 0, 0.0, D.addr(X), mm, 0, len(ps),
                   amap=D.addr(rmap), sAm=mi, bmap=D.addr(_row_maps(dt, dt.nidx_h[ps], mj)), sBm=mj,
                   cmap=D.addr(rmap), sCm=mi)
        out.append(X)
    return assemble_near(dt, out[0], out[1], bases.U, k)


def _gram_chol(dt, Om, ld_om, amap, n, s, nb_):
    torch = _torch()
    f64 = _f64(dt.device)
    G = torch.empty((nb_, n, n), **f64)
    R = torch.zeros_like(G)
    D.gemm(0, 1, n, n, s, 1.0, D.addr(Om), ld_om, 0, D.addr(Om), ld_om, 0, 0.0, D.addr(G), n, n * n, nb_,
           amap=D.addr(amap), sAm=n, bmap=D.addr(amap), sBm=n)
    f = D.cholesky_upper(G, R)
    return R, f


def _cond_estimate(R, f, iters=40):
    """cond(Omega[nbr]) = sigma_max(R) / sigma_min(R) (B B^T = R^T R), the number
    ref/reconstruction.py:256-263 takes from an SVD: sigma_max^2 by power
    iteration on R^T R, 1 / sigma_min^2 by inverse iteration through the two
    triangular solves with R, `iters` steps each (batched over the blocks).
    Both iterations approach their limits from the inside, so this converges
    to the exact ratio from below."""
    torch = _torch()
    nb, n, _ = R.shape
    f64 = _f64(R.device)
    v0 = torch.from_numpy(np.random.default_rng(12345).standard_normal((nb, n, 1))).to(R.device)
    tmp = torch.empty((nb, D.NB, 1), **f64)

    def unit(x):
        return x / torch.linalg.vector_norm(x, dim=1, keepdim=True)

    v = unit(v0.clone())
    w = torch.empty_like(v)
    lam_max = None
    for _ in range(iters):
        D.gemm(0, 0, n, 1, n, 1.0, D.addr(R), n, n * n, D.addr(v), 1, n, 0.0, D.addr(w), 1, n, nb)      # R v
        D.gemm(1, 0, n, 1, n, 1.0, D.addr(R), n, n * n, D.addr(w), 1, n, 0.0, D.addr(v), 1, n, nb)      # R^T R v
        lam_max = torch.linalg.vector_norm(v, dim=1).reshape(-1)
        v = unit(v)
    u = unit(v0.clone())
    lam_inv = None
    for _ in range(iters):
        D.trsm_left(R, u, f, f.inv, upper=True, trans=True, tmp=tmp)     # R^-T u
        D.trsm_left(R, u, f, f.inv, upper=True, trans=False, tmp=tmp)    # R^-1 R^-T u
        lam_inv = torch.linalg.vector_norm(u, dim=1).reshape(-1)
        u = unit(u)
    return torch.sqrt(lam_max * lam_inv).cpu().numpy()


def gaussian_pinv_discrepancy(bundle, bases, cond_limit: float = 1e8):
    """B1 near blocks (ref/reconstruction.py:266-307), ragged blocks supported."""
    torch = _torch()
    dt = bases.dt
    mm = dt.m_max
    k = bases.rank
    s = bundle.s
    P = dt.n_pairs
    f64 = _f64(dt.device)
    sizes = dt.sizes
    st = _lib.stream_handle()
    nbr_n = np.array([int(sizes[dt.nidx_h[dt.nptr_h[i]:dt.nptr_h[i + 1]]].sum()) for i in range(dt.b)])
    side_out = []
    for Om_d, Ysrc, Ub, label in ((bundle._omega_d, bundle.Y, bases.U, "neighbor"),
                                  (bundle._psi_d, bundle.Z, bases.V, "neighbor adjoint")):
        pieces = torch.empty((P, mm, mm), **f64)      # per pair (i, j): x_i[:, cols of j], padded
        for n, m in sorted(set(zip(nbr_n.tolist(), sizes.tolist()))):
            n, m = int(n), int(m)
            blk = np.flatnonzero((nbr_n == n) & (sizes == m))
            nb_ = len(blk)
            maps = np.stack([np.concatenate([np.arange(dt.off_h[j], dt.off_h[j + 1])
                                             for j in dt.nidx_h[dt.nptr_h[i]:dt.nptr_h[i + 1]]]) for i in blk])
            amap = torch.from_numpy(maps.astype(np.int32)).to(dt.device)
            R, f = _gram_chol(dt, Om_d, Om_d.stride(0), amap, n, s, nb_)
            D.check_status(f, "Gram of Omega[nbr]")
            cond = _cond_estimate(R, f)
            for bi, c in zip(blk, cond):
                if c > cond_limit:
                    warnings.warn(f"block {bi}: {label} test-matrix stack has condition {c:.2e}")
            rmap = _row_maps(dt, blk, m)
            # Py = Y_i - U_i (U_i^T Y_i)   (m x s)
            Py = torch.empty((nb_, m, s), **f64)
            _lib.call("ublr_gather", D.addr(Ysrc), Ysrc.stride(0), 0, D.addr(rmap), m, m, s, 0, 0, D.addr(Py), s,
                      m * s, nb_, st)
            _perp_rows(dt, Ub, k, Py, s, m, blk, np.arange(nb_))
            # x = Py B^T G^-1 = ((Py B^T) R^-1) R^-T
            X = torch.empty((nb_, m, n), **f64)
            D.gemm(0, 1, m, n, s, 1.0, D.addr(Py), s, m * s, D.addr(Om_d), Om_d.stride(0), 0, 0.0, D.addr(X), n,
                   m * n, nb_, bmap=D.addr(amap), sBm=n)
            D.trsm_right_upper(X, R, f, torch.empty((nb_, m, D.NB), **f64))
            Xt = torch.empty((nb_, n, m), **f64)
            _lib.call("ublr_gather", D.addr(X), n, m * n, None, 0, m, n, 0, 1, D.addr(Xt), m, n * m, nb_, st)
            D.trsm_left(R, Xt, f, f.inv, upper=True, trans=False, tmp=torch.empty((nb_, D.NB, m), **f64))
            # split x_i^T (n x m) by neighbour: pair p = nptr[i] + t holds the
            # rows of neighbour t (at the stacked offset of its block), transposed
            for li, i in enumerate(blk):
                at = 0
                for t in range(dt.nptr_h[i + 1] - dt.nptr_h[i]):
                    p = int(dt.nptr_h[i] + t)
                    mj = int(sizes[dt.nidx_h[p]])
                    _lib.call("ublr_gather", D.addr(Xt, li * n * m + at * m), m, 0, None, 0, mj, m, 0, 1,
                              D.addr(pieces, p * mm * mm), mm, 0, 1, st)
                    at += mj
        side_out.append(pieces)
    return assemble_near(dt, side_out[0], side_out[1], bases.U, k)


def pinv_core(op, bundle, bases, B_flat, p: int, stream, max_width=None):
    """C = U^T (Y - B Omega) (V^T Omega)^+ (ref/reconstruction.py:379-421).
    Returns (core K x K device tensor, columns added). Ragged blocks supported."""
    from .reconstruction import blockwise_lt_x
    torch = _torch()
    dt = bases.dt
    mm = dt.m_max
    k = bases.rank
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
            device_apply(inner, dt.perm, D.addr(Of, s), L, extra, D.addr(Yf, s), L, dt.device)
        else:
            Yf[:, s:] = dt.to_perm_rows(inner.apply(dt.from_perm_rows(Of[:, s:])))
    # Rf = Y - B Omega, accumulated by neighbour slot t (no two writers per row
    # block in one launch), near blocks read from the padded per-pair layout
    if (dt.sizes == mm).all():
        Bp = B_flat
    else:
        Bp = torch.zeros(dt.n_pairs * mm * mm, **f64)
        _lib.call("ublr_pairs_pad", D.addr(B_flat), D.addr(dt.b_off), D.addr(dt.pair_i), D.addr(dt.nidx),
                  D.addr(dt.off), dt.n_pairs, mm, D.addr(Bp), 1, st)
    slot = np.arange(dt.n_pairs) - dt.nptr_h[dt.pair_i_h]
    for (t, mi, mj), ps in _slot_groups(dt, slot):
        amap = _imap(dt, ps.astype(np.int64) * mm, mi)
        bmap = _row_maps(dt, dt.nidx_h[ps], mj)
        cmap = _row_maps(dt, dt.pair_i_h[ps], mi)
        D.gemm(0, 0, mi, L, mj, -1.0, D.addr(Bp), mm, 0, D.addr(Of), L, 0, 1.0, D.addr(Yf), L, 0, len(ps),
               amap=D.addr(amap), sAm=mi, bmap=D.addr(bmap), sBm=mj, cmap=D.addr(cmap), sCm=mi)
    # V^T Omega and U^T (Y - B Omega): K x L, block rows of k_i
    VtO = torch.empty((K, L), **f64)
    LHS = torch.empty((K, L), **f64)
    blockwise_lt_x(dt, bases.V, k, Of, VtO)
    blockwise_lt_x(dt, bases.U, k, Yf, LHS)
    del Of, Yf
    core = lstsq_right(LHS, VtO)
    return core, extra


def _slot_groups(dt, slot):
    """Pairs grouped by (neighbour slot, m_i, m_j)."""
    out = {}
    for p in range(dt.n_pairs):
        i, j = int(dt.pair_i_h[p]), int(dt.nidx_h[p])
        out.setdefault((int(slot[p]), int(dt.sizes[i]), int(dt.sizes[j])), []).append(p)
    return [(kk, np.asarray(v)) for kk, v in sorted(out.items())]


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
