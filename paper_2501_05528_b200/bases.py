"""Step I of compression on the GPU: per-block bases from sketches.

Mirrors ref/bases.py (BlockBases, SketchBundle, tagging_bases, ...). All
arrays live in HBM in the block-contiguous layout of `DeviceTess`; the
reference-shaped numpy views (`u_blocks`, `omega`, ...) are materialised
lazily, only when a caller asks for them.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .linalg import RandomStream, device_normals
from .operators import CountingOperator, unwrap
from .tessellation import Tessellation, device_tess


def _torch():
    import torch
    return torch


class BlockBases:
    """ref/bases.py:49-65; U, V are N x k device tensors (permuted rows)."""

    def __init__(self, dt, U, V, rank, method, sketch_columns):
        self.dt = dt
        self.U = U
        self.V = V
        self.rank = rank
        self.method = method
        self.sketch_columns = sketch_columns
        self.effective_ranks = dt.ranks(rank).astype(np.int64)

    @property
    def total_rank(self) -> int:
        return int(self.effective_ranks.sum())

    def rank_offsets(self) -> np.ndarray:
        return np.concatenate(([0], np.cumsum(self.effective_ranks)))

    def _blocks(self, M):
        h = M.cpu().numpy()
        off = self.dt.off_h
        return [h[off[i]:off[i + 1], :self.effective_ranks[i]].copy() for i in range(self.dt.b)]

    @property
    def u_blocks(self) -> list:
        return self._blocks(self.U)

    @property
    def v_blocks(self) -> list:
        return self._blocks(self.V)


class SketchBundle:
    """ref/bases.py:30-46; device tensors, host views on demand."""

    def __init__(self, kind, dt, s, Y, Z, G=None, H=None, tagging=None, group_cols=None,
                 omega_d=None, psi_d=None, block_cols=None):
        self.kind = kind
        self.dt = dt
        self.tess = dt.tess
        self.s = s
        self.Y, self.Z = Y, Z
        self.G, self.H = G, H
        self.tagging = tagging
        self.group_cols = group_cols
        self.block_cols = block_cols
        self._omega_d, self._psi_d = omega_d, psi_d

    def omega_device(self):
        if self._omega_d is None:
            self._omega_d = assemble_tagged(self.dt, self.tagging.entries, self.G, self.group_cols)
        return self._omega_d

    def psi_device(self):
        if self._psi_d is None:
            self._psi_d = assemble_tagged(self.dt, self.tagging.entries, self.H, self.group_cols)
        return self._psi_d

    @property
    def omega(self) -> np.ndarray:
        return self.dt.from_perm_rows(self.omega_device())

    @property
    def psi(self) -> np.ndarray:
        return self.dt.from_perm_rows(self.psi_device())

    @property
    def y(self) -> np.ndarray:
        return self.dt.from_perm_rows(self.Y)

    @property
    def z(self) -> np.ndarray:
        return self.dt.from_perm_rows(self.Z)

    def _blocks(self, M):
        h = M.cpu().numpy()
        off = self.dt.off_h
        return [h[off[i]:off[i + 1]].copy() for i in range(self.dt.b)]

    @property
    def g_blocks(self):
        return None if self.G is None else self._blocks(self.G)

    @property
    def h_blocks(self):
        return None if self.H is None else self._blocks(self.H)


def assemble_tagged(dt, T_entries, G, gc):
    """Omega (permuted rows): block i, group c holds T[i, c] G_i
    (ref/bases.py:126-137). Only used when a black-box host operator needs
    the explicit test matrix; the GPU operators never materialise it."""
    torch = _torch()
    T = torch.as_tensor(np.asarray(T_entries), dtype=torch.float64, device=G.device)
    blk = torch.repeat_interleave(torch.arange(dt.b, device=G.device), torch.as_tensor(dt.sizes, device=G.device))
    return (T[blk][:, :, None] * G[:, None, :]).reshape(G.shape[0], -1).contiguous()


def _bill(op, a_cols, astar_cols):
    if isinstance(op, CountingOperator):
        if a_cols:
            op.ledger.record_apply(a_cols)
        if astar_cols:
            op.ledger.record_adjoint(astar_cols)


def draw_test_blocks(dt, stream: RandomStream, side: int, cols: int):
    """G_i = gaussian(m_i, cols, stream.child(side, i)) for every block, as one
    N x cols device tensor (ref/bases.py:163-168)."""
    torch = _torch()
    out = torch.empty((dt.n, cols), dtype=torch.float64, device=dt.device)
    specs = [(stream.child(side, i), int(dt.sizes[i]), cols, int(dt.off_h[i]) * cols, cols, None)
             for i in range(dt.b)]
    return device_normals(specs, out)


def tagged_sketch(op, dt, T_dev, T_entries, G, H, gc):
    """Y = A Omega, Z = A^* Psi for the tagged test matrices; returns (Y, Z)."""
    torch = _torch()
    inner = unwrap(op)
    ell = T_entries.shape[1]
    s = ell * gc
    stream = _lib.stream_handle()
    if hasattr(inner, "device_op"):
        Y = torch.empty((dt.n, s), dtype=torch.float64, device=dt.device)
        Z = torch.empty((dt.n, s), dtype=torch.float64, device=dt.device)
        if getattr(inner, "symmetric", False):
            _lib.call("ublr_sketch_tagged_pair", inner.device_op(dt.perm), _lib.ptr(dt.off), dt.b,
                      _lib.ptr(T_dev), ell, _lib.ptr(G), _lib.ptr(H), gc, gc, _lib.ptr(Y), _lib.ptr(Z), s, stream)
        else:
            _lib.call("ublr_sketch_tagged", inner.device_op(dt.perm), _lib.ptr(dt.off), dt.b, _lib.ptr(T_dev),
                      ell, _lib.ptr(G), gc, gc, _lib.ptr(Y), s, stream)
            _lib.call("ublr_sketch_tagged", inner.device_op(dt.perm, adjoint=True), _lib.ptr(dt.off), dt.b,
                      _lib.ptr(T_dev), ell, _lib.ptr(H), gc, gc, _lib.ptr(Z), s, stream)
        return Y, Z
    # black-box host operator: explicit test matrices through its apply
    om = assemble_tagged(dt, T_entries, G, gc)
    ps = assemble_tagged(dt, T_entries, H, gc)
    Y = dt.to_perm_rows(inner.apply(dt.from_perm_rows(om)))
    Z = dt.to_perm_rows(inner.apply_adjoint(dt.from_perm_rows(ps)))
    return Y, Z


def block_bases_from_tagged(dt, Y, Z, Z_dev, ell, gc, k):
    """U_i, V_i = leading Q of the z^(i)-combined samples (K4)."""
    torch = _torch()
    s = ell * gc
    U = torch.zeros((dt.n, k), dtype=torch.float64, device=dt.device)
    V = torch.zeros((dt.n, k), dtype=torch.float64, device=dt.device)
    stream = _lib.stream_handle()
    kq = max(1, min(k, dt.m_max))
    for src, dst in ((Y, U), (Z, V)):
        _lib.call("ublr_block_qr", _lib.ptr(src), s, 0, _lib.ptr(Z_dev), ell, gc, None, _lib.ptr(dt.off), dt.b,
                  kq, _lib.ptr(dst), k, stream, dt.m_max)
    return U, V


def tagging_bases(op, tess: Tessellation, k: int, p: int, plan, stream: RandomStream,
                  group_cols: int | None = None, extra_samples: bool = False):
    """ref/bases.py:140-204 on the GPU. Returns (BlockBases, SketchBundle)."""
    torch = _torch()
    if extra_samples:
        raise NotImplementedError("extra_samples (ref/bases.py:177-182) is not on the B200 hot path (SURVEY F12)")
    _lib.require_device()
    dt = device_tess(tess, torch.device("cuda"))
    r = k + p
    gc = r if group_cols is None else group_cols
    T_entries = plan.matrix.entries
    ell = T_entries.shape[1]
    s = ell * gc
    if k > dt.m_max and k > 0:
        pass  # every block takes the identity basis (ref/bases.py:80-82)
    G = draw_test_blocks(dt, stream, 0, gc)
    H = draw_test_blocks(dt, stream, 1, gc)
    T_dev = torch.from_numpy(np.ascontiguousarray(T_entries)).to(dt.device)
    Z_dev = torch.from_numpy(np.ascontiguousarray(plan.Z)).to(dt.device)
    _bill(op, s, s)
    Y, Z = tagged_sketch(op, dt, T_dev, T_entries, G, H, gc)
    U, V = block_bases_from_tagged(dt, Y, Z, Z_dev, ell, gc, k)
    bases = BlockBases(dt, U, V, k, "tag", (s, s))
    bundle = SketchBundle("tag", dt, s, Y, Z, G=G, H=H, tagging=plan.matrix, group_cols=gc)
    return bases, bundle
