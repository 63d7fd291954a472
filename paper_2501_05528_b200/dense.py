"""Host drivers of the blocked batched dense kernels (csrc/dense.cu).

Right-looking blocked algorithms over batches of equal-size matrices; every
flop runs in the sm_100a kernels (GEMM with DMMA, nb x nb panel
factorisations in shared memory). All matrices are row-major CUDA float64
tensors of shape (batch, rows, cols) unless stated.
"""

from __future__ import annotations

import numpy as np

from . import _lib

NB = 64


def _torch():
    import torch
    return torch


def _dense(*ts):
    for t in ts:
        if t is not None and not t.is_contiguous():
            raise ValueError("dense kernels take contiguous row-major (batch, rows, cols) tensors")


def addr(t, offset_elems=0) -> int:
    return int(t.data_ptr()) + 8 * int(offset_elems)


def gemm(ta, tb, M, N, K, alpha, A, lda, sA, B, ldb, sB, beta, C, ldc, sC, batch,
         amap=0, sAm=0, bmap=0, sBm=0, cmap=0, sCm=0):
    """Pointer-level batched GEMM: A, B, C (and the optional row maps) are
    addresses (ints)."""
    _lib.call("ublr_gemm_batched", int(ta), int(tb), int(M), int(N), int(K), float(alpha), A, int(lda), int(sA),
              amap or None, int(sAm), B, int(ldb), int(sB), bmap or None, int(sBm), float(beta), C, int(ldc), int(sC),
              cmap or None, int(sCm), int(batch), _lib.stream_handle())


class Factors:
    """Diagonal-block inverses kept for the blocked triangular solves."""

    def __init__(self, n, nb, batch, device):
        torch = _torch()
        self.n, self.nb, self.batch = n, nb, batch
        self.blocks = [(j0, min(nb, n - j0)) for j0 in range(0, n, nb)]
        self.inv = torch.zeros((len(self.blocks), batch, nb, nb), dtype=torch.float64, device=device)
        self.inv2 = None  # second set (U^-1 for LU)


def _split(w, nb):
    """Left part of a recursive split of w columns, on an nb boundary."""
    nblk = -(-w // nb)
    return nb * ((nblk + 1) // 2)


def _syrk_upper(M, K, alpha, A, lda, sA, beta, C, ldc, sC, batch):
    _lib.call("ublr_syrk_upper_batched", int(M), int(K), float(alpha), A, int(lda), int(sA), float(beta), C,
              int(ldc), int(sC), int(batch), _lib.stream_handle())


def _trsm_rec(T, n, f, inv_set, j0, a, X, ldx, Y, ldy, N, batch, lower_unit):
    """Y = op(T11)^-1 X for the diagonal range [j0, j0 + a) of T (n x n,
    batch stride n*n): lower_unit -> T11 is the unit-lower L of an LU; else
    T11 = R^T with R upper (Cholesky). X and Y are addresses inside n x n
    matrices (batch stride n*n) of the range's rows, N columns. Recursive: the
    off-diagonal update is one GEMM with K = a/2 at the top; the nb x nb leaves
    multiply by the stored diagonal-block inverses. X is consumed; Y must not
    alias it."""
    nn = n * n
    if a <= f.nb:
        bi = j0 // f.nb
        gemm(0 if lower_unit else 1, 0, a, N, a, 1.0, addr(inv_set[bi]), a, a * a, X, ldx, nn, 0.0, Y, ldy, nn,
             batch)
        return
    h = _split(a, f.nb)
    _trsm_rec(T, n, f, inv_set, j0, h, X, ldx, Y, ldy, N, batch, lower_unit)
    if lower_unit:   # X_bot -= L[j0+h:j0+a, j0:j0+h] Y_top
        gemm(0, 0, a - h, N, h, -1.0, addr(T, (j0 + h) * n + j0), n, nn, Y, ldy, nn, 1.0, X + 8 * h * ldx, ldx, nn,
             batch)
    else:            # X_bot -= R[j0:j0+h, j0+h:j0+a]^T Y_top
        gemm(1, 0, a - h, N, h, -1.0, addr(T, j0 * n + j0 + h), n, nn, Y, ldy, nn, 1.0, X + 8 * h * ldx, ldx, nn,
             batch)
    _trsm_rec(T, n, f, inv_set, j0 + h, a - h, X + 8 * h * ldx, ldx, Y + 8 * h * ldy, ldy, N, batch, lower_unit)


def cholesky_upper(G, R, nb=NB):
    """G_b = R_b^T R_b (G overwritten as workspace, only its upper triangle is
    read; R zero-initialised by the caller). Recursive: chol(G11); R12 =
    R11^-T G12; G22 -= R12^T R12 (upper tiles, K = half the range); chol(G22)
    — the updates are large-K GEMMs instead of a rank-64 update per panel.
    Returns Factors with R_jj^-1 of the nb x nb diagonal blocks. Raises
    LinAlgError (check_status) if not SPD."""
    torch = _torch()
    _dense(G, R)
    batch, n, _ = G.shape
    f = Factors(n, nb, batch, G.device)
    status = torch.zeros(1, dtype=torch.int32, device=G.device)
    nn = n * n

    def rec(j0, w):
        if w <= nb:
            bi = j0 // nb
            _lib.call("ublr_potrf_diag", addr(G), n, nn, j0, w, addr(R), n, nn, addr(f.inv[bi]), addr(status),
                      batch, _lib.stream_handle())
            return
        a = _split(w, nb)
        rec(j0, a)
        _trsm_rec(R, n, f, f.inv, j0, a, addr(G, j0 * n + j0 + a), n, addr(R, j0 * n + j0 + a), n, w - a, batch,
                  lower_unit=False)
        _syrk_upper(w - a, a, -1.0, addr(R, j0 * n + j0 + a), n, nn, 1.0, addr(G, (j0 + a) * n + j0 + a), n, nn,
                    batch)
        rec(j0 + a, w - a)

    rec(0, n)
    f.status = status
    return f


def lu_sign(W, LU, D, nb=NB, R=None):
    """No-pivot LU of W + diag(D) with D_jj = sign(w_jj) picked at pivot time
    (W overwritten). LU holds unit-L (strict lower) and U. Returns Factors
    with L_jj^-1 (inv) and U_jj^-1 (inv2) of the nb x nb diagonal blocks.

    With an upper-triangular R (batch x n x n) the factored matrix is
    W + diag(D) R instead (row j of D R joins when j becomes the pivot row):
    for W = -B1^T and R the Cholesky factor of B B^T this is (D - Q_top) R,
    whose L is the L of D - Q_top (bn null space).

    Recursive on columns: LU of the left half (all rows), U12 = L11^-1 W12,
    W22 -= L21 U12 (K = half the range), LU of the right half."""
    torch = _torch()
    _dense(W, LU, D, R)
    batch, n, _ = W.shape
    f = Factors(n, nb, batch, W.device)
    f.inv2 = torch.zeros_like(f.inv)
    status = torch.zeros(1, dtype=torch.int32, device=W.device)
    nn = n * n

    def rec(j0, w):
        if w <= nb:
            bi = j0 // nb
            if R is None:
                _lib.call("ublr_lu_sign_diag", addr(W), n, nn, j0, w, addr(LU), n, nn, addr(f.inv[bi]),
                          addr(f.inv2[bi]), addr(D), n, addr(status), batch, _lib.stream_handle())
            else:
                # panel only (n = j0 + w); the rows' D R12 to the right in one parallel pass
                _lib.call("ublr_lu_sign_diag_r", addr(W), n, nn, j0, w, addr(LU), n, nn, addr(f.inv[bi]),
                          addr(f.inv2[bi]), addr(D), n, addr(status), addr(R), n, nn, j0 + w, batch,
                          _lib.stream_handle())
                if j0 + w < n:
                    _lib.call("ublr_add_scaled_rows", addr(W, j0 * n + j0 + w), n, nn, addr(R, j0 * n + j0 + w), n,
                              nn, addr(D, j0), n, w, n - j0 - w, batch, _lib.stream_handle())
            if j0 + w < n:   # L21 = W21 U11^-1 for every row below
                gemm(0, 0, n - j0 - w, w, w, 1.0, addr(W, (j0 + w) * n + j0), n, nn, addr(f.inv2[bi]), w, w * w,
                     0.0, addr(LU, (j0 + w) * n + j0), n, nn, batch)
            return
        a = _split(w, nb)
        rec(j0, a)
        _trsm_rec(LU, n, f, f.inv, j0, a, addr(W, j0 * n + j0 + a), n, addr(LU, j0 * n + j0 + a), n, w - a, batch,
                  lower_unit=True)
        gemm(0, 0, n - j0 - a, w - a, a, -1.0, addr(LU, (j0 + a) * n + j0), n, nn, addr(LU, j0 * n + j0 + a), n, nn,
             1.0, addr(W, (j0 + a) * n + j0 + a), n, nn, batch)
        rec(j0 + a, w - a)

    rec(0, n)
    f.status = status
    return f


def trsm_right_upper(X, R, f: Factors, tmp):
    """X_b <- X_b R_b^-1 in place (X: batch x rows x n, R upper n x n).
    tmp: (batch, rows, nb) scratch. Recursive on columns: Y1 = X1 R11^-1,
    X2 -= Y1 R12 (one GEMM with K = half the range), Y2 = X2 R22^-1; the
    nb-column leaves multiply by the stored diagonal-block inverses."""
    batch, rows, n = X.shape
    nn = n * n
    sx = rows * n
    st = tmp.shape[1] * tmp.shape[2]

    def rec(j0, a):
        if a <= f.nb:
            bi = j0 // f.nb
            _lib.call("ublr_gather", addr(X, j0), n, sx, None, 0, rows, a, 0, 0, addr(tmp), tmp.shape[2], st, batch,
                      _lib.stream_handle())
            gemm(0, 0, rows, a, a, 1.0, addr(tmp), tmp.shape[2], st, addr(f.inv[bi]), a, a * a,
                 0.0, addr(X, j0), n, sx, batch)
            return
        h = _split(a, f.nb)
        rec(j0, h)
        gemm(0, 0, rows, a - h, h, -1.0, addr(X, j0), n, sx, addr(R, j0 * n + j0 + h), n, nn, 1.0,
             addr(X, j0 + h), n, sx, batch)
        rec(j0 + h, a - h)

    rec(0, n)


def trsm_left(T, X, f: Factors, inv_set, upper: bool, trans: bool, tmp):
    """X_b <- op(T_b)^-1 X_b in place, op = transpose if `trans`.
    T: batch x n x n (only the triangle selected by `upper` is read; the
    diagonal blocks come from the stored inverses `inv_set` of T's own
    diagonal blocks). X: batch x n x w. tmp: batch x nb x w.
    Recursive on rows (forward for a lower op(T), backward for an upper one):
    the off-diagonal update is one GEMM with K = half the range, so the
    flops run at large-K GEMM rates instead of rank-nb panel updates."""
    batch, n, w = X.shape
    nn = n * n
    sx = n * w
    stt = tmp.shape[1] * tmp.shape[2]
    eff_lower = (not upper) != trans  # lower-triangular after op

    def leaf(j0, jb):
        bi = j0 // f.nb
        _lib.call("ublr_gather", addr(X, j0 * w), w, sx, None, 0, jb, w, 0, 0, addr(tmp), w, stt, batch,
                  _lib.stream_handle())
        gemm(1 if trans else 0, 0, jb, w, jb, 1.0, addr(inv_set[bi]), jb, jb * jb, addr(tmp), w, stt,
             0.0, addr(X, j0 * w), w, sx, batch)

    def update(r0, r1, c0, c1):
        # X[r0:r1] -= op(T)[r0:r1, c0:c1] X[c0:c1]; op(T)[r, c] = T[r, c] or T[c, r]
        if not trans:
            gemm(0, 0, r1 - r0, w, c1 - c0, -1.0, addr(T, r0 * n + c0), n, nn, addr(X, c0 * w), w, sx,
                 1.0, addr(X, r0 * w), w, sx, batch)
        else:
            gemm(1, 0, r1 - r0, w, c1 - c0, -1.0, addr(T, c0 * n + r0), n, nn, addr(X, c0 * w), w, sx,
                 1.0, addr(X, r0 * w), w, sx, batch)

    def rec(j0, a):
        if a <= f.nb:
            leaf(j0, a)
            return
        h = _split(a, f.nb)
        if eff_lower:
            rec(j0, h)
            update(j0 + h, j0 + a, j0, j0 + h)
            rec(j0 + h, a - h)
        else:
            rec(j0 + h, a - h)
            update(j0, j0 + h, j0 + h, j0 + a)
            rec(j0, h)

    rec(0, n)


def check_status(f: Factors, what: str):
    if int(f.status.item()) != 0:
        raise np.linalg.LinAlgError(f"{what}: factorisation broke down (matrix not positive definite / singular)")
