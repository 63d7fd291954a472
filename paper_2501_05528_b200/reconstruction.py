"""Compressed uBLR format and the compression pipelines on the GPU.

Mirrors ref/reconstruction.py (UniformBLR, direct_core,
structured_identity_discrepancy, compress_type_a / _b, compress,
CompressionReport, relative_error). Step functions keep the reference's
signatures; their work runs in the CUDA kernels of `csrc/` through the C ABI.
"""

from __future__ import annotations

import time
from collections.abc import Mapping
from dataclasses import dataclass

import numpy as np

from . import _lib
from .bases import BlockBases, block_nullification_bases, draw_test_pair, naive_bases, tagging_bases
from .linalg import RandomStream, device_normals
from .operators import CountingOperator, DifferenceOperator, LinearOperatorHandle, counting_wrapper, unwrap
from .tagging import DegenerateTagsError, make_tagging_matrix, plan_tagging
from .tessellation import BoxColoring, Tessellation, color_boxes, device_tess

METHOD_IDS = {("A", "bn"): "A1", ("A", "tag"): "A2", ("A", "naive"): "A3", ("B", "bn"): "B1", ("B", "tag"): "B2"}


def _torch():
    import torch
    return torch


class UniformBLR:
    """U C V* + B over a tessellation (ref/reconstruction.py:50-132).

    Device storage: U, V are N x k (permuted rows), `core_d` is K x K, B is
    one flat buffer of near blocks in neighbour-CSR order (b_off). The
    reference's fields (`u_blocks`, `v_blocks`, `core`, `b_blocks`) are
    host views built on demand."""

    def __init__(self, tess, rank, U, V, core_d, B_d, dt, metadata=None):
        self.tess = tess
        self.rank = rank
        self.dt = dt
        self.U, self.V = U, V
        self.core_d = core_d
        self.B_d = B_d
        self.effective_ranks = dt.ranks(rank).astype(np.int64)
        self.metadata = metadata or {}
        self._host = {}

    # --- reference-shaped views -------------------------------------------
    @property
    def n(self) -> int:
        return self.tess.n_points

    @property
    def shape(self) -> tuple:
        return (self.n, self.n)

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
        if "u" not in self._host:
            self._host["u"] = self._blocks(self.U)
        return self._host["u"]

    @property
    def v_blocks(self) -> list:
        if "v" not in self._host:
            self._host["v"] = self._blocks(self.V)
        return self._host["v"]

    @property
    def core(self) -> np.ndarray:
        if "core" not in self._host:
            self._host["core"] = self.core_d.cpu().numpy()
        return self._host["core"]

    @property
    def b_blocks(self) -> dict:
        if "B" not in self._host:
            flat = self.B_d.cpu().numpy()
            dt = self.dt
            out = {}
            for p in range(dt.n_pairs):
                i, j = int(dt.pair_i_h[p]), int(dt.nidx_h[p])
                out[(i, j)] = flat[dt.b_off_h[p]:dt.b_off_h[p + 1]].reshape(dt.sizes[i], dt.sizes[j])
            self._host["B"] = out
        return self._host["B"]

    def to_host(self) -> dict:
        """Copy U, V, core and the near blocks to pinned host memory in one
        asynchronous pass (one stream sync); returns numpy arrays in the
        device layout (permuted rows)."""
        torch = _torch()
        out = {}
        for name, t in (("U", self.U), ("V", self.V), ("core", self.core_d), ("B", self.B_d)):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t, non_blocking=True)
            out[name] = h
        torch.cuda.current_stream().synchronize()
        return {k: v.numpy() for k, v in out.items()}

    @property
    def storage_entries(self) -> int:
        return int(2 * sum(self.dt.sizes * self.effective_ranks) + self.total_rank ** 2 + self.dt.b_off_h[-1])

    # --- products -----------------------------------------------------------
    def apply_device(self, Xd, adjoint=False):
        """A_hat X on permuted rows (N x w CUDA tensor)."""
        return blr_apply(self, Xd, adjoint)

    def apply(self, X):
        X = np.asarray(X, dtype=float)
        vec = X.ndim == 1
        X2 = X.reshape(-1, 1) if vec else X
        out = self.dt.from_perm_rows(self.apply_device(self.dt.to_perm_rows(X2)))
        return out.ravel() if vec else out

    def apply_adjoint(self, X):
        X = np.asarray(X, dtype=float)
        vec = X.ndim == 1
        X2 = X.reshape(-1, 1) if vec else X
        out = self.dt.from_perm_rows(self.apply_device(self.dt.to_perm_rows(X2), adjoint=True))
        return out.ravel() if vec else out

    def to_dense(self) -> np.ndarray:
        return self.apply(np.eye(self.n))


def blr_apply(rep: UniformBLR, Xd, adjoint=False):
    """Blockwise U C V^T X + B X, or the adjoint (ref/reconstruction.py:93-119),
    through the C-ABI kernel `ublr_blr_apply` (ragged blocks supported)."""
    torch = _torch()
    dt = rep.dt
    n, w = Xd.shape
    Xd = Xd.contiguous()
    K = rep.total_rank
    roff_h, roff = dt.roff(rep.rank)
    out = torch.empty((n, w), dtype=torch.float64, device=Xd.device)
    lib = _lib.load()
    work = torch.empty(int(lib.ublr_blr_apply_workspace_bytes(K, w)) // 8 + 1, dtype=torch.float64,
                       device=Xd.device)
    core = rep.core_d if K > 0 else work
    _lib.call("ublr_blr_apply", _lib.ptr(rep.U), _lib.ptr(rep.V), rep.U.stride(0), _lib.ptr(core), K,
              _lib.ptr(rep.B_d), _lib.ptr(dt.b_off), _lib.ptr(dt.off), _lib.ptr(roff), _lib.ptr(dt.nptr),
              _lib.ptr(dt.nidx), _lib.ptr(dt.tpair), dt.b, _lib.ptr(Xd), w, w, 1 if adjoint else 0,
              _lib.ptr(out), w, _lib.ptr(work), _lib.stream_handle())
    return out


def relative_error(op, rep: UniformBLR, iterations: int = 20, stream: RandomStream | None = None) -> float:
    """ref/reconstruction.py:160-177 (power method on A - A_hat and on A)."""
    from .linalg import gaussian  # host draws keep the reference's start vectors
    torch = _torch()
    stream = stream or RandomStream(0)
    if op.shape != rep.shape:
        raise ValueError(f"shape mismatch: {op.shape} vs {rep.shape}")
    dt = rep.dt
    inner = unwrap(op)

    def a_apply(Xd, adj):
        if hasattr(inner, "apply_device"):
            return inner.apply_device(Xd, dt.perm, adjoint=adj and not getattr(inner, "symmetric", False))
        f = inner.apply_adjoint if adj else inner.apply
        return dt.to_perm_rows(f(dt.from_perm_rows(Xd)))

    def power(fwd, adj, st):
        if iterations < 1:
            raise ValueError("iterations must be >= 1")
        v = dt.to_perm_rows(gaussian(dt.n, 1, st))
        nv = torch.linalg.vector_norm(v)
        if float(nv) == 0.0:
            return 0.0
        v = v / nv
        est = 0.0
        for _ in range(iterations):
            w = fwd(v)
            est = float(torch.linalg.vector_norm(w))
            if est == 0.0:
                return 0.0
            v = adj(w)
            v = v / torch.linalg.vector_norm(v)
        return est

    num = power(lambda X: a_apply(X, False) - rep.apply_device(X),
                lambda X: a_apply(X, True) - rep.apply_device(X, adjoint=True), stream.child(0))
    den = power(lambda X: a_apply(X, False), lambda X: a_apply(X, True), stream.child(1))
    if den == 0.0:
        raise ValueError("operator norm estimate is zero")
    return num / den


@dataclass
class FrobeniusReport:
    """Exact blockwise Frobenius norms (ublr_frob_error / ublr_frob_diff).

    `pair2[i - i0, j]` holds the squared norm of pair (i, j) for the block
    rows i0 <= i < i1 that were evaluated; `ref2` the squared norms of the
    minuend (||A_ij||^2 for an error report, None for a difference)."""
    i0: int
    i1: int
    pair2: np.ndarray
    ref2: np.ndarray | None

    @property
    def fro(self) -> float:
        return float(np.sqrt(self.pair2.sum()))

    @property
    def ref_fro(self) -> float | None:
        return None if self.ref2 is None else float(np.sqrt(self.ref2.sum()))

    @property
    def relative(self) -> float:
        return self.fro / self.ref_fro


def _rep_rows(rep, i0):
    """U / core pointers of a representation, shifted for a block-row shard
    whose arrays start at block row `i0` (rep.row0 / rep.k0)."""
    dt = rep.dt
    r0 = int(dt.off_h[i0]) - int(getattr(rep, "row0", 0))
    return r0, getattr(rep, "k0", 0)


def frobenius_error(op, rep: UniformBLR, i0: int = 0, i1: int | None = None) -> FrobeniusReport:
    """||A - A_hat||_F blockwise and exactly, A generated on the device
    (ublr_frob_error). The BASELINE.json approximation-error gate; the
    reference reports a 20-step power-method spectral estimate instead
    (ref/reconstruction.py:160-177)."""
    torch = _torch()
    dt = rep.dt
    i1 = dt.b if i1 is None else i1
    inner = unwrap(op)
    if not hasattr(inner, "device_op"):
        raise NotImplementedError("frobenius_error needs an operator with a device descriptor")
    roff_h, roff = dt.roff(rep.rank)
    rows = max(i1 - i0, 0)
    err2 = torch.zeros((rows, dt.b), dtype=torch.float64, device=dt.device)
    a2 = torch.zeros_like(err2)
    row0 = int(getattr(rep, "row0", 0))
    k0 = int(getattr(rep, "k0", 0))
    _lib.call("ublr_frob_error", inner.device_op(dt.perm), _lib.ptr(dt.off), _lib.ptr(dt.nptr), _lib.ptr(dt.nidx),
              _lib.ptr(dt.b_off), dt.b, _lib.ptr(roff), int(max(rep.effective_ranks.max(initial=0), 0)),
              _lib.ptr(rep.U) - 8 * row0 * rep.U.stride(0), _lib.ptr(rep.V), rep.U.stride(0),
              _lib.ptr(rep.core_d) - 8 * k0 * rep.core_d.stride(0), rep.core_d.stride(0),
              _lib.ptr(rep.B_d) - 8 * int(getattr(rep, "b0", 0)), i0, i1, _lib.ptr(err2), _lib.ptr(a2),
              _lib.stream_handle())
    return FrobeniusReport(i0, i1, err2.cpu().numpy(), a2.cpu().numpy())


def frobenius_distance(rep1: UniformBLR, rep2: UniformBLR, i0: int = 0, i1: int | None = None) -> FrobeniusReport:
    """||A_hat1 - A_hat2||_F blockwise and exactly (ublr_frob_diff), for two
    representations on the same tessellation."""
    torch = _torch()
    dt = rep1.dt
    if rep2.dt.b != dt.b or not np.array_equal(rep2.dt.off_h, dt.off_h):
        raise ValueError("frobenius_distance: representations on different tessellations")
    i1 = dt.b if i1 is None else i1
    _, roff1 = dt.roff(rep1.rank)
    _, roff2 = rep2.dt.roff(rep2.rank)
    d2 = torch.zeros((max(i1 - i0, 0), dt.b), dtype=torch.float64, device=dt.device)

    def args(rep):
        row0, k0 = int(getattr(rep, "row0", 0)), int(getattr(rep, "k0", 0))
        return (int(max(rep.effective_ranks.max(initial=0), 0)), _lib.ptr(rep.U) - 8 * row0 * rep.U.stride(0),
                _lib.ptr(rep.V), rep.U.stride(0), _lib.ptr(rep.core_d) - 8 * k0 * rep.core_d.stride(0),
                rep.core_d.stride(0), _lib.ptr(rep.B_d) - 8 * int(getattr(rep, "b0", 0)))

    _lib.call("ublr_frob_diff", _lib.ptr(dt.off), _lib.ptr(dt.nptr), _lib.ptr(dt.nidx), _lib.ptr(dt.b_off), dt.b,
              _lib.ptr(roff1), *args(rep1), _lib.ptr(roff2), *args(rep2), i0, i1, _lib.ptr(d2), _lib.stream_handle())
    return FrobeniusReport(i0, i1, d2.cpu().numpy(), None)


# ---------------------------------------------------------------------------
# Type A
# ---------------------------------------------------------------------------

def _groups(dt, k):
    """Blocks grouped by (m_i, k_i) for the batched blockwise GEMMs:
    [(m, ki, blocks)]."""
    ranks = dt.ranks(k)
    out = {}
    for i in range(dt.b):
        out.setdefault((int(dt.sizes[i]), int(ranks[i])), []).append(i)
    return [(m, ki, np.asarray(bl)) for (m, ki), bl in sorted(out.items())]


def _rows_map(starts, width):
    torch = _torch()
    rows = np.asarray(starts, dtype=np.int64)[:, None] + np.arange(width)[None, :]
    return torch.from_numpy(rows.astype(np.int32)).cuda()


def blockwise_lt_x(dt, L, k, X, out):
    """out[roff_i : roff_i + k_i, :] = L_i^T X[rows_i, :] for every block
    (L = U or V, N x ld; X N x w; out K x w), batched per (m_i, k_i) group on
    ublr_gemm_batched with row maps (ragged blocks supported)."""
    from . import dense as D
    roff_h, _ = dt.roff(k)
    w = X.shape[1]
    for m, ki, bl in _groups(dt, k):
        if ki == 0:
            continue
        rmap = _rows_map(dt.off_h[bl], m)
        D.gemm(1, 0, ki, w, m, 1.0, D.addr(L), L.stride(0), 0, D.addr(X), X.stride(0), 0, 0.0, D.addr(out),
               out.stride(0), 0, len(bl), amap=D.addr(rmap), sAm=m, bmap=D.addr(rmap), sBm=m,
               cmap=D.addr(_rows_map(roff_h[bl], ki)), sCm=ki)


def blockwise_l_y(dt, L, k, Yk, out, alpha=1.0, beta=0.0):
    """out[rows_i, :] = alpha L_i Yk[roff_i : roff_i + k_i, :] + beta out[rows_i, :]."""
    from . import dense as D
    roff_h, _ = dt.roff(k)
    w = Yk.shape[1]
    for m, ki, bl in _groups(dt, k):
        rmap = _rows_map(dt.off_h[bl], m)
        if ki == 0:
            if beta != 1.0:
                for i in bl:
                    out[dt.off_h[i]:dt.off_h[i + 1]].mul_(beta)
            continue
        D.gemm(0, 0, m, w, ki, alpha, D.addr(L), L.stride(0), 0, D.addr(Yk), Yk.stride(0), 0, beta, D.addr(out),
               out.stride(0), 0, len(bl), amap=D.addr(rmap), sAm=m, bmap=D.addr(_rows_map(roff_h[bl], ki)), sBm=ki,
               cmap=D.addr(rmap), sCm=m)


def _direct_core_host_op(inner, dt, bases, core):
    """direct_core for a black-box host operator: V_dense (N x K, block
    diagonal) goes through op.apply as in ref/reconstruction.py:189-197; the
    projections C_i = U_i^T (A V)[rows_i] run on the device."""
    torch = _torch()
    k = bases.rank
    roff_h, _ = dt.roff(k)
    K = int(roff_h[-1])
    Vd = torch.zeros((dt.n, K), dtype=torch.float64, device=dt.device)
    ranks = dt.ranks(k)
    for j in range(dt.b):
        Vd[dt.off_h[j]:dt.off_h[j + 1], roff_h[j]:roff_h[j] + ranks[j]] = bases.V[dt.off_h[j]:dt.off_h[j + 1], :ranks[j]]
    AV = dt.to_perm_rows(np.asarray(inner.apply(dt.from_perm_rows(Vd)), dtype=np.float64))
    del Vd
    blockwise_lt_x(dt, bases.U, k, AV, core)
    return core


def direct_core(op, tess: Tessellation, bases: BlockBases):
    """C = U^T (A V) (ref/reconstruction.py:185-198); device K x K tensor."""
    torch = _torch()
    dt = bases.dt
    k = bases.rank
    K = bases.total_rank
    roff_h, roff = dt.roff(k)
    core = torch.empty((K, K), dtype=torch.float64, device=dt.device)
    if isinstance(op, CountingOperator):
        op.ledger.record_apply(K)
    inner = unwrap(op)
    if K == 0:
        return core
    if not hasattr(inner, "device_op"):
        return _direct_core_host_op(inner, dt, bases, core)
    if dt.m_max <= FUSED_NEAR_M_MAX and min(k, dt.m_max) <= FUSED_NEAR_K_MAX and dt.pair_of is not None:
        # small blocks: the colour-probe near field (phase III) comes out of the
        # same pass over A (ublr_coupling_nearfield); structured_identity_discrepancy
        # returns it for this core
        B = torch.empty(max(int(dt.b_off_h[-1]), 1), dtype=torch.float64, device=dt.device)
        _lib.call("ublr_coupling_nearfield", inner.device_op(dt.perm), _lib.ptr(dt.off), _lib.ptr(roff), dt.b, k,
                  _lib.ptr(bases.U), _lib.ptr(bases.V), bases.U.stride(0), _lib.ptr(core), K, _lib.ptr(dt.cptr),
                  _lib.ptr(dt.cidx), dt.n_colours, dt.m_max, _lib.ptr(dt.pair_of), _lib.ptr(dt.nidx),
                  _lib.ptr(dt.b_off), _lib.ptr(B), _lib.stream_handle(), 0, dt.b)
        bases.fused_near = (core, _versions(core, bases), inner, B[:int(dt.b_off_h[-1])])
        return core
    _lib.call("ublr_coupling", inner.device_op(dt.perm), _lib.ptr(dt.off), _lib.ptr(roff), dt.b, k,
              _lib.ptr(bases.U), _lib.ptr(bases.V), bases.U.stride(0), _lib.ptr(core), K, _lib.stream_handle(),
              dt.m_max, 0, dt.b)
    return core


def _versions(core, bases):
    """In-place modification counters of the fused near field's inputs."""
    return (core._version, bases.U._version, bases.V._version)


FUSED_NEAR_M_MAX = 64   # ublr_coupling_nearfield limits
FUSED_NEAR_K_MAX = 32


def _check_coloring(tess, colors):
    """ref/reconstruction.py:214-221: no two blocks of one neighbourhood share a colour."""
    from .tagging import _neighbour_csr
    colors = np.asarray(colors, dtype=np.int64)
    ptr, idx = _neighbour_csr(tess)
    seg = np.repeat(np.arange(tess.b, dtype=np.int64), np.diff(ptr))
    key = seg * (int(colors.max(initial=0)) + 1) + colors[idx]
    if np.unique(key).size != key.size:
        for i in range(tess.b):
            nc = colors[tess.neighbor_lists[i]]
            if len(set(nc.tolist())) != len(nc):
                raise ValueError(f"invalid coloring: two same-color probes collide in the neighborhood of block {i}")


def _colour_layout(dt, cols):
    """Device colour arrays (colour per block, member CSR) of a caller-supplied
    colouring, cached per colouring on the device tessellation."""
    torch = _torch()
    key = ("colours", cols.tobytes())
    hit = dt.rng_records.get(key)
    if hit is None:
        n = int(cols.max()) + 1
        order = np.argsort(cols, kind="stable")
        cptr = np.concatenate(([0], np.cumsum(np.bincount(cols, minlength=n)))).astype(np.int32)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dt.device)  # noqa: E731
        hit = (t(cols.astype(np.int32)), t(cptr), t(order.astype(np.int32)), n)
        dt.rng_records[key] = hit
    return hit


def _structured_identity_host_op(inner, tess, bases, core, cols):
    """structured_identity_discrepancy for a black-box host operator: one
    identity probe per colour through op.apply (ref/reconstruction.py:227-243);
    V^T probe, C (V^T probe) and the subtraction of U_i (C V^T probe)[rows_i]
    run on the device, and the near blocks are cut out of the residual
    (including the same-colour leak)."""
    from . import dense as D
    torch = _torch()
    dt = bases.dt
    k = bases.rank
    K = bases.total_rank
    sizes = dt.sizes
    B = torch.empty(max(int(dt.b_off_h[-1]), 1), dtype=torch.float64, device=dt.device)
    pair = {(int(i), int(j)): q for q, (i, j) in enumerate(zip(dt.pair_i_h, dt.nidx_h))}
    for c in range(int(cols.max()) + 1):
        members = np.flatnonzero(cols == c)
        if members.size == 0:
            continue
        mc = int(sizes[members].max())
        probe = np.zeros((dt.n, mc))
        for j in members:
            probe[tess.blocks[j], np.arange(sizes[j])] = 1.0
        R = dt.to_perm_rows(np.asarray(inner.apply(probe), dtype=np.float64))
        if K > 0:
            P = dt.to_perm_rows(probe)
            VtP = torch.empty((K, mc), dtype=torch.float64, device=dt.device)
            blockwise_lt_x(dt, bases.V, k, P, VtP)
            CV = torch.empty((K, mc), dtype=torch.float64, device=dt.device)
            D.gemm(0, 0, K, mc, K, 1.0, D.addr(core), core.stride(0), 0, D.addr(VtP), mc, 0, 0.0, D.addr(CV), mc, 0,
                   1)
            blockwise_l_y(dt, bases.U, k, CV, R, alpha=-1.0, beta=1.0)
        for j in members:
            for i in tess.neighbor_lists[j]:
                q = pair[(int(i), int(j))]
                B[int(dt.b_off_h[q]):int(dt.b_off_h[q + 1])].view(int(sizes[i]), int(sizes[j])).copy_(
                    R[dt.off_h[i]:dt.off_h[i + 1], :sizes[j]])
    return B[:int(dt.b_off_h[-1])]


def structured_identity_discrepancy(op, tess: Tessellation, bases: BlockBases, core, coloring: BoxColoring):
    """Near blocks from colour probes, with the reference's same-colour leak
    (ref/reconstruction.py:201-244). Returns a flat device buffer
    of near blocks in neighbour-CSR order."""
    torch = _torch()
    dt = bases.dt
    cols = np.asarray(coloring.colors)
    checked = tess._device.get("coloring_checked")
    if checked is None or not np.array_equal(checked, cols):
        _check_coloring(tess, cols)          # pure function of (tess, colours): validated once
        tess._device["coloring_checked"] = cols.copy()
    k = bases.rank
    K = bases.total_rank
    roff_h, roff = dt.roff(k)
    sizes = dt.sizes
    ncol = int(cols.max()) + 1 if cols.size else 0
    if isinstance(op, CountingOperator):
        op.ledger.record_apply(int(sum(sizes[cols == c].max() for c in range(ncol) if (cols == c).any())))
    inner = unwrap(op)
    if not hasattr(inner, "device_op"):
        return _structured_identity_host_op(inner, tess, bases, core, cols)
    custom = not np.array_equal(cols, dt.colours_h)
    fused = getattr(bases, "fused_near", None)
    if not custom and fused is not None and fused[0] is core and fused[1] == _versions(core, bases) and fused[2] is inner:
        return fused[3]   # computed with this core by direct_core's fused pass
    B = torch.empty(int(dt.b_off_h[-1]), dtype=torch.float64, device=dt.device)
    lib = _lib.load()
    ws_bytes = int(lib.ublr_nearfield_workspace_bytes(dt.n_pairs, max(k, 1), dt.m_max))
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=dt.device)
    if K == 0:
        core = torch.zeros((1, 1), dtype=torch.float64, device=dt.device)
    colours_d, cptr_d, cidx_d, n_colours = (_colour_layout(dt, cols) if custom else
                                            (dt.colours, dt.cptr, dt.cidx, dt.n_colours))
    _lib.call("ublr_nearfield_colour", inner.device_op(dt.perm), _lib.ptr(dt.off), _lib.ptr(roff), dt.b, k,
              _lib.ptr(bases.U), _lib.ptr(bases.V), bases.U.stride(0), _lib.ptr(core), max(K, 1),
              _lib.ptr(colours_d), _lib.ptr(cptr_d), _lib.ptr(cidx_d), n_colours, dt.m_max,
              _lib.ptr(dt.pair_i), _lib.ptr(dt.nidx), dt.n_pairs, _lib.ptr(dt.b_off), _lib.ptr(B),
              _lib.ptr(ws), ws_bytes, _lib.stream_handle())
    return B


# ---------------------------------------------------------------------------
# Reports and pipelines
# ---------------------------------------------------------------------------

@dataclass
class CompressionReport:
    """ref/reconstruction.py:429-463."""
    method: str
    config: dict
    matvecs: dict
    times_s: dict
    relative_error: float | None
    storage_entries: int
    aspect_ratios: dict | None = None

    @property
    def matvecs_total(self) -> int:
        return sum(v["A"] + v["Astar"] for v in self.matvecs.values())

    def phase_total(self, phase: str) -> int:
        e = self.matvecs.get(phase, {"A": 0, "Astar": 0})
        return e["A"] + e["Astar"]

    def to_dict(self) -> dict:
        return {"method": self.method, "config": self.config, "matvecs": self.matvecs,
                "matvecs_total": self.matvecs_total,
                "times_s": {k: float(f"{v:.3g}") for k, v in self.times_s.items()},
                "relative_error": self.relative_error, "storage_entries": self.storage_entries,
                "aspect_ratios": self.aspect_ratios}


def _quantiles(sorted_vals: np.ndarray, qs) -> list:
    """np.quantile(..., method="linear") on sorted data, restated (same
    virtual index and two-sided lerp as numpy, so the same bits) without
    numpy's per-call overhead."""
    n = sorted_vals.size
    out = []
    for q in qs:
        v = n * q + (1.0 - q) - 1.0
        lo = int(np.floor(v))
        lo = min(max(lo, 0), n - 1)
        hi = min(lo + 1, n - 1)
        t = v - np.floor(v)
        a, b = float(sorted_vals[lo]), float(sorted_vals[hi])
        d = b - a
        out.append(b - d * (1.0 - t) if t >= 0.5 else a + d * t)
    return out


def _ratio_summary(values: np.ndarray) -> dict:
    fin = np.sort(values[np.isfinite(values)])
    if fin.size == 0:
        return {"count": 0}
    q1, med, q3 = _quantiles(fin, (0.25, 0.5, 0.75))
    return {"count": int(fin.size), "min": float(fin[0]), "q1": float(q1),
            "median": float(med), "q3": float(q3), "max": float(fin[-1])}


def _base_config(tess, k, p, stream, **extra) -> dict:
    cfg = {"N": tess.n_points, "b": tess.b, "m": tess.max_block_size, "k": k, "p": p, "d": tess.dim,
           "seed": stream.seed}
    cfg.update(extra)
    return cfg


class PhaseTimes(Mapping):
    """Per-phase seconds (ref/reconstruction.py:524-551 `times_s`), measured as
    CUDA-event spans on the compression stream. Recording never blocks the
    host; the events are resolved (one synchronisation) on first read."""

    def __init__(self):
        self._events = {}
        self._values = None

    def _record(self, name, e0, e1):
        self._events[name] = (e0, e1)
        self._values = None

    def _resolve(self):
        if self._values is None:
            vals = {}
            for name, (e0, e1) in self._events.items():
                e1.synchronize()
                vals[name] = e0.elapsed_time(e1) / 1e3
            self._values = vals
        return self._values

    def __getitem__(self, key):
        return self._resolve()[key]

    def __iter__(self):
        return iter(self._resolve())

    def __len__(self):
        return len(self._events)

    def __repr__(self):
        return repr(dict(self._resolve()))


class _PhaseTimer:
    """CUDA events around a phase on the current stream (no host sync)."""

    def __init__(self, times: PhaseTimes, name):
        self.times, self.name = times, name

    def __enter__(self):
        self.e0 = _torch().cuda.Event(enable_timing=True)
        self.e0.record(_lib.current_stream())

    def __exit__(self, *exc):
        e1 = _torch().cuda.Event(enable_timing=True)
        e1.record(_lib.current_stream())
        self.times._record(self.name, self.e0, e1)


class _Lazy:
    """A value computed on first call (the host tagging draw, deferred until
    the sketch of its device twin has been launched)."""

    def __init__(self, fn):
        self._fn, self._done, self._v = fn, False, None

    def __call__(self):
        if not self._done:
            self._v, self._done = self._fn(), True
        return self._v


def _stream_scoped(fn):
    """Run a compressor with the CUDA stream handle captured once (_lib.stream_scope)."""
    import functools

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        with _lib.stream_scope():
            return fn(*args, **kwargs)
    return wrapped


@_stream_scoped
def compress_type_a(op, tess, k, p=10, method="tag", stream=None, distribution="gaussian", extra_cols=0,
                    optimize=False, extra_samples=False, max_tag_redraws=5, compute_error=True,
                    error_iterations=20):
    """ref/reconstruction.py:498-583 on the GPU."""
    stream = stream or RandomStream(0)
    _lib.require_device()
    cop = counting_wrapper(op)
    times, plan = PhaseTimes(), None
    with _PhaseTimer(times, "I"), cop.ledger.phase("I"):
        if method == "tag":
            # the test blocks are drawn on the GPU while the host draws the
            # tagging matrix; the sketch of the policy's first draw runs while
            # the host evaluates the plan
            test_pair = None
            if not extra_samples:
                # gaussian tagging: T is drawn in the same launch (the host draws the same bits below)
                ell = 3 ** tess.dim + 1 + extra_cols
                # (not with optimize: the device null vectors are the base ones)
                tag = ((stream.child(1).child(0), ell) if distribution == "gaussian" and tess.b >= ell
                       and not optimize else (None, 0))
                test_pair = draw_test_pair(device_tess(tess, _torch().device("cuda")), stream.child(0), k + p, *tag)
            first = _Lazy(lambda: make_tagging_matrix(tess.b, tess.dim, extra_cols, distribution,
                                                      stream.child(1).child(0)))
            bases, bundle = tagging_bases(
                cop, tess, k, p,
                lambda: plan_tagging(tess, extra_cols, distribution, stream.child(1), optimize=optimize,
                                     max_redraws=max_tag_redraws, device="auto", first=first()),
                stream.child(0), extra_samples=extra_samples, first=first, test_pair=test_pair, defer_plan=True)
            plan = bundle.plan
        elif method == "bn":
            bases, _ = block_nullification_bases(cop, tess, k, p, stream.child(0))
        elif method == "naive":
            bases, _ = naive_bases(cop, tess, k, p, stream.child(0))
        else:
            raise ValueError(f"unknown step-I method {method!r}")
    with _PhaseTimer(times, "II"), cop.ledger.phase("II"):
        core = direct_core(cop, tess, bases)
    with _PhaseTimer(times, "III"):
        coloring = color_boxes(tess)
        with cop.ledger.phase("III"):
            B = structured_identity_discrepancy(cop, tess, bases, core, coloring)
    if method == "tag" and plan is None:
        # the bases were built from the device draw of the first tagging
        # matrix and phases II-III are queued behind them; the host evaluates
        # the redraw policy now, overlapping that GPU work, and everything is
        # recomputed (without billing the ledger twice) if it redrew
        plan, redo = bundle.resolve_plan()
        bundle.resolve_plan = None
        bundle.plan, bundle.tagging = plan, plan.matrix
        if redo is not None:
            (bases.U, bases.V), bundle.Y, bundle.Z = redo
            inner = unwrap(cop)
            core = direct_core(inner, tess, bases)
            B = structured_identity_discrepancy(inner, tess, bases, core, coloring)
    rep = UniformBLR(tess, k, bases.U, bases.V, core, B, bases.dt, {"method": METHOD_IDS[("A", method)]})
    rel = relative_error(op, rep, error_iterations, stream.child(9)) if compute_error else None
    aspect, ell = None, None
    if plan is not None:
        ell = plan.matrix.n_cols
        aspect = {"base": _ratio_summary(plan.rho_base), "draws": plan.attempts}
        if plan.rho_optimized is not None:
            aspect["optimized"] = _ratio_summary(plan.rho_optimized)
    report = CompressionReport(
        method=METHOD_IDS[("A", method)],
        config=_base_config(tess, k, p, stream, ell=ell, distribution=distribution if method == "tag" else None,
                            extra_cols=extra_cols if method == "tag" else None, optimize=optimize),
        matvecs=cop.ledger.to_dict(), times_s=times, relative_error=rel,
        storage_entries=rep.storage_entries, aspect_ratios=aspect)
    return rep, report


@_stream_scoped
def compress_type_b(op, tess, k, p=10, method="bn", stream=None, distribution="gaussian", optimize=False,
                    max_tag_redraws=5, compute_error=True, error_iterations=20, max_width=None):
    """ref/reconstruction.py:586-677 on the GPU: bases, near field from the
    reused sketches (phase III), then the core by least squares (phase II)."""
    from .tagging import b2_denominators_ok
    from .typeb import gaussian_pinv_discrepancy, pinv_core, tagging_pinv_discrepancy

    stream = stream or RandomStream(0)
    if method not in ("bn", "tag"):
        raise ValueError("type B supports methods 'bn' and 'tag'")
    _lib.require_device()
    cop = counting_wrapper(op)
    times, plan = PhaseTimes(), None
    with _PhaseTimer(times, "I"), cop.ledger.phase("I"):
        if method == "bn":
            bases, bundle = block_nullification_bases(cop, tess, k, p, stream.child(0))
        else:
            first = make_tagging_matrix(tess.b, tess.dim, 0, distribution, stream.child(1).child(0))
            bases, bundle = tagging_bases(
                cop, tess, k, p,
                lambda: plan_tagging(tess, 0, distribution, stream.child(1), optimize=optimize,
                                     max_redraws=max_tag_redraws, device="auto", extra_check=lambda T: b2_denominators_ok(T, tess), first=first),
                stream.child(0), group_cols=tess.max_block_size + p, first=first, compensated=True)
            plan = bundle.plan
    with _PhaseTimer(times, "III"), cop.ledger.phase("III"):
        if method == "bn":
            B = gaussian_pinv_discrepancy(bundle, bases)
        else:
            B = tagging_pinv_discrepancy(bundle, bases)
    with _PhaseTimer(times, "II"), cop.ledger.phase("II"):
        core, _ = pinv_core(cop, bundle, bases, B, p, stream.child(2), max_width=max_width)
    rep = UniformBLR(tess, k, bases.U, bases.V, core, B, bases.dt, {"method": METHOD_IDS[("B", method)]})
    rel = relative_error(op, rep, error_iterations, stream.child(9)) if compute_error else None
    aspect, ell = None, None
    if plan is not None:
        ell = plan.matrix.n_cols
        aspect = {"base": _ratio_summary(plan.rho_base), "draws": plan.attempts}
        if plan.rho_optimized is not None:
            aspect["optimized"] = _ratio_summary(plan.rho_optimized)
    report = CompressionReport(
        method=METHOD_IDS[("B", method)],
        config=_base_config(tess, k, p, stream, ell=ell, distribution=distribution if method == "tag" else None,
                            extra_cols=None, optimize=optimize),
        matvecs=cop.ledger.to_dict(), times_s=times, relative_error=rel,
        storage_entries=rep.storage_entries, aspect_ratios=aspect)
    return rep, report


def compress(op, tess, k, method_id: str = "A2", **kwargs):
    """ref/reconstruction.py:680-687."""
    for (family, basis), mid in METHOD_IDS.items():
        if mid == method_id:
            fn = compress_type_a if family == "A" else compress_type_b
            return fn(op, tess, k, method=basis, **kwargs)
    raise ValueError(f"unknown method id {method_id!r}; expected one of {sorted(METHOD_IDS.values())}")
