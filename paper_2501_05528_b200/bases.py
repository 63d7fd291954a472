"""Step I of compression on the GPU: per-block bases from sketches.

Mirrors ref/bases.py (BlockBases, SketchBundle, tagging_bases, ...). All
arrays live in HBM in the block-contiguous layout of `DeviceTess`; the
reference-shaped numpy views (`u_blocks`, `omega`, ...) are materialised
lazily, only when a caller asks for them.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib
from .linalg import RandomStream, device_normals
from .operators import CountingOperator, device_apply, unwrap
from .tagging import DEVICE_PLAN_MIN_B
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


class TestPair:
    """(G, H, T) drawn into one buffer by draw_test_pair with a tagging
    stream. The launches that follow need only the device addresses
    (G_ptr, H_ptr, T_ptr); the torch views are built on first access, after
    those launches are queued (each view op costs microseconds of host time
    on the compression's critical path)."""

    def __init__(self, buf, n, cols, b, tag_cols):
        self.buf, self.n, self.cols, self.b, self.tag_cols = buf, n, cols, b, tag_cols
        self.G_ptr = int(buf.data_ptr())
        self.H_ptr = self.G_ptr + 8 * n * cols
        self.T_ptr = self.G_ptr + 16 * n * cols
        self._views = None

    def views(self):
        if self._views is None:
            n2 = 2 * self.n * self.cols
            GH = self.buf[:n2].view(2, self.n, self.cols)
            self._views = (GH[0], GH[1], self.buf[n2:].view(self.b, self.tag_cols))
        return self._views

    def __len__(self):
        return 3

    def __getitem__(self, i):
        return self.views()[i]

    def __iter__(self):
        return iter(self.views())


def draw_test_pair(dt, stream: RandomStream, cols: int, tag_stream: RandomStream | None = None, tag_cols: int = 0):
    """(G, H) with G_i = gaussian(m_i, cols, stream.child(0, i)) and
    H_i = ...child(1, i) (ref/bases.py:163-168), drawn in ONE launch set into
    a (2, N, cols) buffer. With `tag_stream`, the same launch also draws the
    gaussian tagging matrix T = gaussian(b, tag_cols, tag_stream)
    (ref/tagging.py:61-91) on the device and a TestPair (G, H, T) is returned: the host
    draws the same bits with numpy for its planning, and the sketch can be
    launched without waiting for a host-to-device copy of T."""
    from .linalg import launch_normals, rng_launch_record

    torch = _torch()
    n2 = 2 * dt.n * cols
    tn = dt.b * tag_cols if tag_stream is not None else 0
    buf = torch.empty(n2 + tn, dtype=torch.float64, device=dt.device)
    ck = ("test_pair", stream.seed, tuple(stream.key), cols,
          None if tag_stream is None else (tag_stream.seed, tuple(tag_stream.key), tag_cols))
    rec = dt.rng_records.get(ck)
    if rec is None:
        b = dt.b
        keys = [tuple(stream.key) + (side, i) for side in (0, 1) for i in range(b)]
        rows = np.concatenate([dt.sizes, dt.sizes]).astype(np.int64)
        offs = np.concatenate([dt.off_h[:-1].astype(np.int64) * cols,
                               dt.n * cols + dt.off_h[:-1].astype(np.int64) * cols])
        if tag_stream is None:
            suffix = np.stack([np.repeat(np.arange(2), b), np.tile(np.arange(b), 2)], axis=1)  # (side, i)
            rec = rng_launch_record(stream.seed, stream.key, rows, cols, offs, cols, None, dt.device, suffix=suffix)
        else:
            if tag_stream.seed != stream.seed:
                raise ValueError("tagging and test-block streams must share the seed")
            rec = rng_launch_record(stream.seed, keys + [tuple(tag_stream.key)], np.append(rows, b),
                                    np.append(np.full(2 * b, cols), tag_cols), np.append(offs, n2),
                                    np.append(np.full(2 * b, cols), tag_cols), None, dt.device)
        if len(dt.rng_records) > 16:
            dt.rng_records.clear()
        dt.rng_records[ck] = rec
    launch_normals(rec, buf)
    if tag_stream is None:
        GH = buf[:n2].view(2, dt.n, cols)
        return GH[0], GH[1]
    return TestPair(buf, dt.n, cols, dt.b, tag_cols)


STAGED_SKETCH_MIN_ROWS = 16384   # below, one fused launch beats per-strip launches


def staged_sketch_workspace(inner, dt, gc, nrows, ell):
    """(tensor, bytes) for ublr_sketch_tagged_staged, or None when the fused
    entry points should be used: symmetric kernel operators with even n and
    even block offsets (16-byte aligned A chunks), ell <= 10, and a strip that
    fills the SMs within a third of the free memory (capped at 4 GB unless a
    single column tile needs a whole wave of row tiles, as a c5 shard does)."""
    torch = _torch()
    if os.environ.get("UBLR_SKETCH_STAGED", "1") == "0":
        return None
    if getattr(inner, "kind", None) not in ("log", "inv") or not getattr(inner, "symmetric", False):
        return None
    if ell > 10 or dt.n % 2 or gc % 2 or nrows < STAGED_SKETCH_MIN_ROWS or (dt.off_h % 2).any():
        return None
    lib = _lib.load()
    free, _ = torch.cuda.mem_get_info(dt.device)
    ncols = 2 * gc
    ct = -(-ncols // (64 if ncols <= 64 else 128))
    if ct < 2:
        # one column tile (a c5 shard: 128 columns): every entry of A is used
        # once, and writing + reading the strip costs more HBM time than the
        # evaluation inside the kernel does (measured 1,771 against 1,448 ms)
        return None
    want = max(4 << 30, -(-148 // ct) * 32 * dt.n * 8)
    nbytes = min(want, free // 3) // 16 * 16
    if int(lib.ublr_sketch_tagged_staged_rows(dt.n, ncols, nrows, nbytes)) < 32:
        return None
    return torch.empty(nbytes // 8, dtype=torch.float64, device=dt.device), nbytes


def tagged_sketch(op, dt, T_dev, T_entries, G, H, gc, out=None, ell=None, compensated=False):
    """Y = A Omega, Z = A^* Psi for the tagged test matrices; returns (Y, Z)
    (into `out` = (Y, Z) when given). T_entries (host) is needed only by a
    black-box operator. `compensated`: the fold over column blocks recovers
    its rounding errors (ublr_sketch_tagged_comp; type B, where the sketch's
    rounding noise is divided by small projected tags)."""
    torch = _torch()
    inner = unwrap(op)
    ell = T_entries.shape[1] if ell is None else ell
    s = ell * gc
    stream = _lib.stream_handle()
    if hasattr(inner, "device_op"):
        if out is not None:
            Y, Z = out
        else:
            Y = torch.empty((dt.n, s), dtype=torch.float64, device=dt.device)
            Z = torch.empty((dt.n, s), dtype=torch.float64, device=dt.device)
        staged = staged_sketch_workspace(inner, dt, gc, dt.n, ell)
        if staged is not None:
            _lib.call("ublr_sketch_tagged_staged", inner.device_op(dt.perm), _lib.ptr(dt.off), dt.b, _lib.ptr(T_dev),
                      ell, _lib.ptr(G), _lib.ptr(H), gc, gc, _lib.ptr(Y), _lib.ptr(Z), s, 0, dt.n,
                      1 if compensated else 0, _lib.ptr(staged[0]), staged[1], stream)
        elif compensated and ell <= 10:
            if getattr(inner, "symmetric", False):
                _lib.call("ublr_sketch_tagged_comp", inner.device_op(dt.perm), _lib.ptr(dt.off), dt.b,
                          _lib.ptr(T_dev), ell, _lib.ptr(G), _lib.ptr(H), gc, gc, _lib.ptr(Y), _lib.ptr(Z), s, 0, dt.n,
                          stream)
            else:
                _lib.call("ublr_sketch_tagged_comp", inner.device_op(dt.perm), _lib.ptr(dt.off), dt.b,
                          _lib.ptr(T_dev), ell, _lib.ptr(G), None, gc, gc, _lib.ptr(Y), None, s, 0, dt.n, stream)
                _lib.call("ublr_sketch_tagged_comp", inner.device_op(dt.perm, adjoint=True), _lib.ptr(dt.off), dt.b,
                          _lib.ptr(T_dev), ell, _lib.ptr(H), None, gc, gc, _lib.ptr(Z), None, s, 0, dt.n, stream)
        elif getattr(inner, "symmetric", False):
            _lib.call("ublr_sketch_tagged_pair", inner.device_op(dt.perm), _lib.ptr(dt.off), dt.b,
                      _lib.ptr(T_dev), ell, _lib.ptr(G), _lib.ptr(H), gc, gc, _lib.ptr(Y), _lib.ptr(Z), s, 0, dt.n,
                      stream)
        else:   # both sides in one launch (A, A^T descriptors)
            _lib.call("ublr_sketch_tagged_two", inner.device_op(dt.perm), inner.device_op(dt.perm, adjoint=True),
                      _lib.ptr(dt.off), dt.b, _lib.ptr(T_dev), ell, _lib.ptr(G), _lib.ptr(H), gc, gc, _lib.ptr(Y),
                      _lib.ptr(Z), s, 0, dt.n, stream)
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
    # every column is written unless some block has fewer than k points
    alloc = torch.empty if k < int(dt.sizes.min()) else torch.zeros
    U = alloc((dt.n, k), dtype=torch.float64, device=dt.device)
    V = alloc((dt.n, k), dtype=torch.float64, device=dt.device)
    stream = _lib.stream_handle()
    kq = max(1, min(k, dt.m_max))
    _lib.call("ublr_block_qr_pair", _lib.ptr(Y), _lib.ptr(Z), s, _lib.ptr(Z_dev), ell, gc, _lib.ptr(dt.off), dt.b,
              kq, _lib.ptr(U), _lib.ptr(V), k, stream, dt.m_max)
    return U, V


NULLVEC_DEVICE_MAX_ELL = 32   # ublr_null_vectors_device
_PLAN_WORKER = None


def _plan_worker():
    """One persistent worker thread for the host tagging plan (tagging_bases
    with defer_plan)."""
    global _PLAN_WORKER
    if _PLAN_WORKER is None:
        from concurrent.futures import ThreadPoolExecutor
        _PLAN_WORKER = ThreadPoolExecutor(max_workers=1, thread_name_prefix="ublr-plan")
    return _PLAN_WORKER


def tagging_bases(op, tess: Tessellation, k: int, p: int, plan, stream: RandomStream,
                  group_cols: int | None = None, extra_samples: bool = False, first=None, test_pair=None,
                  defer_plan: bool = False, compensated: bool = False):
    """ref/bases.py:140-204 on the GPU. Returns (BlockBases, SketchBundle).
    `compensated`: tagged sketch with the compensated fold (type B; see
    tagged_sketch).

    `plan` is a TaggingPlan, or a zero-argument callable producing one (the
    host redraw policy of ref/tagging.py:306-352) together with `first`, the
    policy's first draw. The sketch depends only on the tagging matrix, not on
    the null vectors, so with a callable the sketch of `first` is launched
    before the host evaluates the plan and runs on the GPU meanwhile; if the
    policy redraws, the sketch is recomputed for the accepted matrix.
    `test_pair` = (G, H) already drawn by draw_test_pair(dt, stream, gc)
    (compress_type_a launches it before the host draws the tagging matrix).
    `defer_plan`: when the bases were built speculatively from the device draw,
    return with bundle.plan = None and leave the host plan evaluation to
    bundle.resolve_plan() (the caller queues more GPU work first); it returns
    (plan, None) if the first draw was accepted, else (plan, ((U, V), Y, Z))
    recomputed for the accepted matrix."""
    torch = _torch()
    _lib.require_device()
    dt = device_tess(tess, torch.device("cuda"))
    r = k + p
    gc = r if group_cols is None else group_cols
    planner = plan if callable(plan) else None
    from .tagging import extra_sample_vectors

    def combine(pl):
        """Per-block combination vectors: the plan's z^(i), or with
        extra_samples the first null direction (tagging.extra_sample_vectors)."""
        return extra_sample_vectors(pl, tess) if extra_samples else pl.Z

    if planner is not None and tess.b >= DEVICE_PLAN_MIN_B:
        # large b: the planner's aspect ratios run on the GPU, so plan before
        # the sketch occupies it (no speculative sketch)
        plan, planner = planner(), None
    first_fn = first if callable(first) else (lambda: first)
    device_T = (planner is not None and test_pair is not None and len(test_pair) == 3
                and hasattr(unwrap(op), "device_op"))
    if device_T:
        # the device draw of the policy's first matrix (draw_test_pair with
        # tag_stream): the sketch is launched before the host has drawn it,
        # from raw addresses (the tensor views are built after the launches)
        T_dev = test_pair.T_ptr
        ell = test_pair.tag_cols
        matrix = None
    else:
        matrix = first_fn() if planner is not None else plan.matrix
        ell = matrix.entries.shape[1]
        T_dev = _lib.h2d(matrix.entries, dt.device)
    T_shape = (dt.b, ell)
    s = ell * gc
    speculative = matrix is None and ell <= NULLVEC_DEVICE_MAX_ELL and not extra_samples
    if speculative:
        ev_drawn = torch.cuda.Event()          # G, H and T drawn: the null vectors need only T
        ev_drawn.record(_lib.current_stream())
    if device_T:
        YZ = torch.empty(2 * dt.n * s, dtype=torch.float64, device=dt.device)
        yp = int(YZ.data_ptr())
        tagged_sketch(op, dt, T_dev, None, test_pair.G_ptr, test_pair.H_ptr, gc, out=(yp, yp + 8 * dt.n * s),
                      ell=ell, compensated=compensated)
    else:
        Y = torch.empty((dt.n, s), dtype=torch.float64, device=dt.device)
        Z = torch.empty((dt.n, s), dtype=torch.float64, device=dt.device)
        G, H = draw_test_pair(dt, stream, gc) if test_pair is None else test_pair[:2]
        Y, Z = tagged_sketch(op, dt, T_dev, None if matrix is None else matrix.entries, G, H, gc, out=(Y, Z),
                             ell=ell, compensated=compensated)
    _bill(op, s, s)
    if device_T:
        YZv = YZ.view(2, dt.n, s)
        Y, Z = YZv[0], YZv[1]
        G, H = test_pair[0], test_pair[1]
    UV = None
    if speculative:
        # speculative bases: the first draw's null vectors on the device (the
        # same bits as the host planner's, csrc/nullvec.cuh) and the block QR,
        # queued behind the sketch; the host evaluates the plan meanwhile and
        # they are recomputed only if the redraw policy rejects the draw. The
        # null vectors run on a side stream beside the sketch (whose grid
        # leaves SMs free), so only the QR waits for both.
        Z_spec = torch.empty((dt.b, ell), dtype=torch.float64, device=dt.device)
        res_spec = torch.empty(dt.b, dtype=torch.float64, device=dt.device)
        side, side_h = _lib.side_stream()
        side.wait_event(ev_drawn)
        _lib.call("ublr_null_vectors_device", _lib.ptr(T_dev), ell, _lib.ptr(dt.nptr), _lib.ptr(dt.nidx), dt.b,
                  _lib.ptr(Z_spec), _lib.ptr(res_spec), side_h, on=side)
        ev_nv = torch.cuda.Event()
        ev_nv.record(side)
        _lib.current_stream().wait_event(ev_nv)
        UV = block_bases_from_tagged(dt, Y, Z, Z_spec, ell, gc, k)
    def evaluate(speculative_matrix):
        """Host draw + redraw policy; (plan, Y, Z, UV) for the accepted matrix."""
        nonlocal Y, Z
        m0 = speculative_matrix
        if m0 is None:
            m0 = first_fn()                  # host draw of the same bits, while the GPU works
            if m0.entries.shape != T_shape:
                raise RuntimeError("device and host tagging draws disagree in shape")
        pl, uv = plan, UV
        if planner is not None:
            pl = planner()                   # host work, overlapping the sketch
            if pl.matrix is not m0:          # redrawn: sketch the accepted matrix
                uv = None
                T_entries = pl.matrix.entries
                Y, Z = tagged_sketch(op, dt, _lib.h2d(T_entries, dt.device), T_entries, G, H, gc,
                                     compensated=compensated)
        if uv is None:
            uv = block_bases_from_tagged(dt, Y, Z, _lib.h2d(combine(pl), dt.device), ell, gc, k)
        return pl, uv

    if defer_plan and UV is not None and planner is not None:
        bases = BlockBases(dt, UV[0], UV[1], k, "tag", (s, s))
        bundle = SketchBundle("tag", dt, s, Y, Z, G=G, H=H, tagging=None, group_cols=gc)
        bundle.plan = None
        def host_plan():                     # worker thread: host numpy + C only, no CUDA calls
            m0 = first_fn()
            if m0.entries.shape != T_shape:
                raise RuntimeError("device and host tagging draws disagree in shape")
            return m0, planner()

        # the host draw and the redraw policy (its C evaluation releases the
        # GIL) run on a worker thread while this thread queues phases II-III
        fut = _plan_worker().submit(host_plan)

        def resolve_plan():
            # (no reference to bundle / bases here: a cycle through this
            # closure would keep the compression's device buffers alive until
            # the cyclic collector runs)
            m0, pl = fut.result()
            if pl.matrix is m0:
                return pl, None
            T_entries = pl.matrix.entries   # redrawn: sketch and bases of the accepted matrix
            Y2, Z2 = tagged_sketch(op, dt, _lib.h2d(T_entries, dt.device), T_entries, G, H, gc,
                                   compensated=compensated)
            uv = block_bases_from_tagged(dt, Y2, Z2, _lib.h2d(combine(pl), dt.device), ell, gc, k)
            return pl, (uv, Y2, Z2)
        bundle.resolve_plan = resolve_plan
        return bases, bundle
    plan, UV = evaluate(matrix)
    U, V = UV
    bases = BlockBases(dt, U, V, k, "tag", (s, s))
    bundle = SketchBundle("tag", dt, s, Y, Z, G=G, H=H, tagging=plan.matrix, group_cols=gc)
    bundle.plan = plan
    return bases, bundle


# ---------------------------------------------------------------------------
# Block nullification (ref/bases.py:68-123)
# ---------------------------------------------------------------------------

def block_nullification_width(tess: Tessellation, r: int) -> int:
    """ref/bases.py:68-75."""
    widest = max(tess.neighbor_row_count(i) for i in range(tess.b))
    return max(r + widest, 3 ** tess.dim * r)


def nullspace_samples(dt, Om, ld_om, col_om, Ysrc, ld_y, s, r, k, S_out, chunk_bytes=40 << 30, nside=1):
    """S_i = Y_i P_k^(i) for every block, P_k^(i) the first k of the r trailing
    null-space columns that null_basis(Omega[nbr(i)], r) returns
    (ref/bases.py:102-110, ref/linalg.py:72-94), without a Householder QR:

      G = B B^T = R^T R (blocked Cholesky),
      LU of (D - Qt_top) R = D R - B[:, :n]^T with D_jj = sign(pivot)
      (Householder reconstruction: reproduces LAPACK's dlarfg reflectors,
      tau in [1, 2]; Qt = B^T R^-1 is never formed),
      M = L^-T U'^-T B[:, E],  P_k = [M ; E_bot] - B^T R^-1 D M

    where B = Omega[nbr(i)] (n x s), Qt = B^T R^-1 and E selects columns
    s-r .. s-r+k-1 (DESIGN.md §bn null space). Blocks with equal
    neighbourhood size n are batched; Omega rows are gathered in place.

    nside = 2 runs both sides of block nullification in the same launches
    (twice the batch, half the launches): Om = [Omega | Psi] and
    Ysrc = [Y | Z] are N x 2s (ld 2s, col_om = 0) and S_out is N x 2 x k.
    Side sigma's row q of a side-by-side pair is the virtual row
    nside * q + sigma of a matrix with leading dimension s (k for S_out), so
    the row maps address both sides without copies."""
    import torch

    from . import dense as D

    dev = dt.device
    if nside == 2 and (ld_om != 2 * s or ld_y != 2 * s or col_om != 0):
        raise ValueError("nullspace_samples(nside=2) needs [Omega | Psi] and [Y | Z] side by side")
    vl_om = s if nside == 2 else ld_om          # leading dimension of the virtual row space
    vl_y = s if nside == 2 else ld_y
    vl_s = k if nside == 2 else S_out.stride(0)

    def vrows(rows, sides):
        """virtual rows (len(sides) * len(blocks), width): side-major batch order."""
        rows = np.asarray(rows, dtype=np.int64)
        return np.concatenate([nside * rows + sg for sg in sides], axis=0)

    sides = list(range(nside))
    om0 = D.addr(Om, col_om)      # Omega side: column offset inside the fused buffer
    sizes = dt.sizes
    nbr_n = np.array([int(sizes[dt.nidx_h[dt.nptr_h[i]:dt.nptr_h[i + 1]]].sum()) for i in range(dt.b)])
    keys = sorted(set(zip(nbr_n.tolist(), sizes.tolist())))
    shared = None
    if (sizes == sizes[0]).all():
        # Omega_j Omega_j'^T once per pair of blocks that share a neighbourhood
        # (13 per block on a 2-D grid instead of 81 per neighbourhood Gram)
        m0 = int(sizes[0])
        pairs = sorted({(min(a, c), max(a, c)) for i in range(dt.b)
                        for a in dt.nidx_h[dt.nptr_h[i]:dt.nptr_h[i + 1]].tolist()
                        for c in dt.nidx_h[dt.nptr_h[i]:dt.nptr_h[i + 1]].tolist()})
        if len(pairs) * nside <= 65535:
            pid = {pq: t for t, pq in enumerate(pairs)}
            pa = np.array(pairs, dtype=np.int64)
            ra = dt.off_h[pa[:, 0]][:, None] + np.arange(m0)[None, :]
            rb = dt.off_h[pa[:, 1]][:, None] + np.arange(m0)[None, :]
            amap_p = torch.from_numpy(vrows(ra, sides).astype(np.int32)).to(dev)
            bmap_p = torch.from_numpy(vrows(rb, sides).astype(np.int32)).to(dev)
            P_all = torch.empty((nside * len(pairs), m0, m0), dtype=torch.float64, device=dev)
            D.gemm(0, 1, m0, m0, s, 1.0, om0, vl_om, 0, om0, vl_om, 0, 0.0, D.addr(P_all), m0, m0 * m0,
                   nside * len(pairs), amap=D.addr(amap_p), sAm=m0, bmap=D.addr(bmap_p), sBm=m0)
            shared = (P_all, pid, len(pairs))
    for n, m in keys:
        n, m = int(n), int(m)
        if s - r < n:
            raise ValueError("block-nullification width too small for a neighbourhood")
        members = np.flatnonzero((nbr_n == n) & (sizes == m))
        per_block = nside * (3 * n * n * 8 + (s + 3 * n) * k * 8)
        ch = max(1, min(len(members), int(chunk_bytes // per_block), 65535 // nside))
        eb = np.zeros((s - n, k))
        eb[np.arange(s - r - n, s - r - n + k), np.arange(k)] = 1.0
        Ebot = torch.from_numpy(eb).to(dev)
        for c0 in range(0, len(members), ch):
            blk = members[c0:c0 + ch]
            nb_ = nside * len(blk)        # batch entries: side-major
            maps = np.stack([np.concatenate([np.arange(dt.off_h[j], dt.off_h[j + 1])
                                             for j in dt.nidx_h[dt.nptr_h[i]:dt.nptr_h[i + 1]]]) for i in blk])
            amap = torch.from_numpy(vrows(maps, sides).astype(np.int32)).to(dev)
            rows = np.stack([np.arange(dt.off_h[i], dt.off_h[i + 1]) for i in blk])
            rmap = torch.from_numpy(vrows(rows, sides).astype(np.int32)).to(dev)
            f64 = dict(dtype=torch.float64, device=dev)
            G = torch.empty((nb_, n, n), **f64)
            R = torch.zeros((nb_, n, n), **f64)
            LU = torch.zeros((nb_, n, n), **f64)
            Dg = torch.zeros((nb_, n), **f64)
            nn = n * n
            # G = B B^T  (B = Omega[nbr]): from the shared neighbour-pair products
            # when blocks are uniform, else gathered in place
            if shared is not None:
                P_all, pid, npairs = shared
                nbl = n // m
                gm = np.empty((nb_, nbl, nbl), dtype=np.int32)
                for sg in sides:
                    for c, i in enumerate(blk):
                        L = dt.nidx_h[dt.nptr_h[i]:dt.nptr_h[i + 1]]
                        for a in range(nbl):
                            for bq in range(nbl):
                                ja, jb = int(L[a]), int(L[bq])
                                t = sg * npairs + (pid[(ja, jb)] if ja <= jb else pid[(jb, ja)])
                                gm[sg * len(blk) + c, a, bq] = t if ja <= jb else -t - 1
                gmap = torch.from_numpy(gm).to(dev)
                _lib.call("ublr_assemble_gram", D.addr(P_all), D.addr(gmap), nbl, m, D.addr(G), nb_,
                          _lib.stream_handle())
            else:
                D.gemm(0, 1, n, n, s, 1.0, om0, vl_om, 0, om0, vl_om, 0, 0.0, D.addr(G), n, nn, nb_,
                       amap=D.addr(amap), sAm=n, bmap=D.addr(amap), sBm=n)
            fC = D.cholesky_upper(G, R)
            # LU of D R - B1^T = (D - Q_top) R  (B1 = B[:, :n]; G is free again)
            W = G
            _lib.call("ublr_gather", om0, vl_om, 0, D.addr(amap), n, n, n, 0, 1, D.addr(W), n, nn, nb_,
                      _lib.stream_handle())
            neg = torch.full((n,), -1.0, **f64)
            _lib.call("ublr_scale_rows", D.addr(W), n, nn, D.addr(neg), 0, n, n, nb_, _lib.stream_handle())
            fL = D.lu_sign(W, LU, Dg, R=R)
            # M = L^-T U^-T R^-T B[:, E] = L^-T U'^-T B[:, E]   (U' = U R)
            Mm = torch.empty((nb_, n, k), **f64)
            _lib.call("ublr_gather", om0, vl_om, 0, D.addr(amap), n, n, k, s - r, 0, D.addr(Mm), k, n * k, nb_,
                      _lib.stream_handle())
            tk = torch.empty((nb_, D.NB, k), **f64)
            D.trsm_left(LU, Mm, fL, fL.inv2, upper=True, trans=True, tmp=tk)
            D.trsm_left(LU, Mm, fL, fL.inv, upper=False, trans=True, tmp=tk)
            # P = [M ; E_bot] - B^T R^-1 (D M)
            P = torch.empty((nb_, s, k), **f64)
            P[:, :n].copy_(Mm)
            P[:, n:].copy_(Ebot)
            DM = Mm
            _lib.call("ublr_scale_rows", D.addr(DM), k, n * k, D.addr(Dg), n, n, k, nb_, _lib.stream_handle())
            D.trsm_left(R, DM, fC, fC.inv, upper=True, trans=False, tmp=tk)
            D.gemm(1, 0, s, k, n, -1.0, om0, vl_om, 0, D.addr(DM), k, n * k, 1.0, D.addr(P), k, s * k, nb_,
                   amap=D.addr(amap), sAm=n)
            # S_i = Y_i P  (rows of block i scattered into S_out)
            D.gemm(0, 0, m, k, s, 1.0, D.addr(Ysrc), vl_y, 0, D.addr(P), k, s * k, 0.0, D.addr(S_out), vl_s, 0, nb_,
                   amap=D.addr(rmap), sAm=m, cmap=D.addr(rmap), sCm=m)
            D.check_status(fC, "Cholesky of Omega[nbr] Omega[nbr]^T")
            D.check_status(fL, "sign-selected LU")


def block_nullification_bases(op, tess: Tessellation, k: int, p: int, stream: RandomStream):
    """ref/bases.py:86-123 on the GPU. Returns (BlockBases, SketchBundle)."""
    torch = _torch()
    _lib.require_device()
    dt = device_tess(tess, torch.device("cuda"))
    r = k + p
    s = block_nullification_width(tess, r)
    n = dt.n
    # Omega | Psi side by side (permuted rows); one numpy stream each, rows in global order
    OP = torch.empty((n, 2 * s), dtype=torch.float64, device=dt.device)
    device_normals([(stream.child(0), n, s, 0, 2 * s, dt.inv), (stream.child(1), n, s, s, 2 * s, dt.inv)], OP)
    _bill(op, s, s)
    inner = unwrap(op)
    YZ = torch.empty((n, 2 * s), dtype=torch.float64, device=dt.device)
    st = _lib.stream_handle()
    if hasattr(inner, "device_op"):
        if getattr(inner, "symmetric", False):
            device_apply(inner, dt.perm, _lib.ptr(OP), 2 * s, 2 * s, _lib.ptr(YZ), 2 * s, dt.device)
        else:
            device_apply(inner, dt.perm, _lib.ptr(OP), 2 * s, s, _lib.ptr(YZ), 2 * s, dt.device)
            device_apply(inner, dt.perm, _lib.ptr(OP) + 8 * s, 2 * s, s, _lib.ptr(YZ) + 8 * s, 2 * s, dt.device,
                         adjoint=True)
    else:
        Yh = inner.apply(dt.from_perm_rows(OP[:, :s]))
        Zh = inner.apply_adjoint(dt.from_perm_rows(OP[:, s:]))
        YZ[:, :s] = dt.to_perm_rows(Yh)
        YZ[:, s:] = dt.to_perm_rows(Zh)
    kq = max(1, min(k, dt.m_max))
    U = torch.zeros((n, max(k, 1)), dtype=torch.float64, device=dt.device)
    V = torch.zeros_like(U)
    Sbuf = torch.zeros((n, 2, kq), dtype=torch.float64, device=dt.device)    # [S_U | S_V] per row
    col0 = torch.zeros(dt.b, dtype=torch.int32, device=dt.device)
    if k < dt.m_max:
        # both sides in the same launches (doubled batches, half the launches)
        nullspace_samples(dt, OP, 2 * s, 0, YZ, 2 * s, s, r, kq, Sbuf, nside=2)
    for side, dst in ((0, U), (1, V)):
        _lib.call("ublr_block_qr", _lib.ptr(Sbuf) + 8 * side * kq, 2 * kq, 1, None, 0, 0, _lib.ptr(col0),
                  _lib.ptr(dt.off), dt.b, kq, _lib.ptr(dst), dst.stride(0), st, dt.m_max)
    bases = BlockBases(dt, U, V, k, "bn", (s, s))
    bundle = SketchBundle("bn", dt, s, YZ[:, :s], YZ[:, s:], omega_d=OP[:, :s], psi_d=OP[:, s:])
    return bases, bundle


def naive_bases(op, tess: Tessellation, k: int, p: int, stream: RandomStream):
    """Blocked randSVD baseline (ref/bases.py:213-260): b zeroed Gaussian
    probes of r columns each, batched into one operator application per side."""
    torch = _torch()
    _lib.require_device()
    dt = device_tess(tess, torch.device("cuda"))
    r = k + p
    n, b = dt.n, dt.b
    w = b * r
    f64 = dict(dtype=torch.float64, device=dt.device)
    OM = torch.empty((n, w), **f64)
    PS = torch.empty((n, w), **f64)
    device_normals([(stream.child(0, i), n, r, i * r, w, dt.inv) for i in range(b)], OM)
    device_normals([(stream.child(1, i), n, r, i * r, w, dt.inv) for i in range(b)], PS)
    # zero the neighbourhood rows of each probe (ref/bases.py:237-239)
    for i in range(b):
        rows = torch.from_numpy(np.concatenate([np.arange(dt.off_h[j], dt.off_h[j + 1])
                                                for j in dt.nidx_h[dt.nptr_h[i]:dt.nptr_h[i + 1]]])).to(dt.device)
        OM[rows, i * r:(i + 1) * r] = 0.0
        PS[rows, i * r:(i + 1) * r] = 0.0
    _bill(op, w, w)
    inner = unwrap(op)
    st = _lib.stream_handle()
    Y = torch.empty((n, w), **f64)
    Z = torch.empty((n, w), **f64)
    if hasattr(inner, "device_op"):
        device_apply(inner, dt.perm, _lib.ptr(OM), w, w, _lib.ptr(Y), w, dt.device)
        device_apply(inner, dt.perm, _lib.ptr(PS), w, w, _lib.ptr(Z), w, dt.device, adjoint=True)
    else:
        Y = dt.to_perm_rows(inner.apply(dt.from_perm_rows(OM)))
        Z = dt.to_perm_rows(inner.apply_adjoint(dt.from_perm_rows(PS)))
    kq = max(1, min(k, dt.m_max))
    U = torch.zeros((n, max(k, 1)), **f64)
    V = torch.zeros_like(U)
    col0 = torch.arange(0, w, r, dtype=torch.int32, device=dt.device)
    for src, dst in ((Y, U), (Z, V)):
        _lib.call("ublr_block_qr", _lib.ptr(src), w, 1, None, 0, 0, _lib.ptr(col0), _lib.ptr(dt.off), b, kq,
                  _lib.ptr(dst), dst.stride(0), st, dt.m_max)
    bases = BlockBases(dt, U, V, k, "naive", (w, w))
    bundle = SketchBundle("naive", dt, w, Y, Z, omega_d=OM, psi_d=PS, block_cols=r)
    return bases, bundle
