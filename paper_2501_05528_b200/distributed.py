"""Block-row sharded type-A tagging compression (config 5).

One process per GPU. Rank r owns a contiguous slab of box rows (block ids
are ordered with grid axis 0 most significant, so a slab is a contiguous
block-id range and a contiguous range of permuted rows). Every rank:

1. plans the tagging matrix and draws ALL test blocks G_j, H_j from the
   shared seed (no communication: the GPU RNG reproduces numpy's streams);
2. sketches its own rows of Y = A Omega and Z = A Psi (A symmetric), and
   forms its U_i, V_i;
3. all-gathers V (N x k, the only collective on the data path: the far-field
   coupling C_ij = U_i^T A_ij V_j needs every V_j, and so does the colour-probe
   leak of the near field, F11);
4. computes its core rows and its near blocks.

`allgather` is pluggable: `torch.distributed.all_gather_into_tensor` (NCCL
over NVLink in production, gloo in the CPU tests) or an in-process
concatenation when ranks are emulated one after another on one GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .bases import _bill, draw_test_pair, staged_sketch_workspace
from .linalg import RandomStream
from .operators import counting_wrapper, unwrap
from .reconstruction import FUSED_NEAR_K_MAX, FUSED_NEAR_M_MAX
from .tagging import plan_tagging
from .tessellation import device_tess


def _torch():
    import torch
    return torch


def _alloc(shape, dtype=None, device=None, zero=False):
    """Device buffers of the shard kernels (a test hook: tests/test_distributed.py
    swaps in a guard-banded allocator to check that the shifted shard
    pointers never write outside their buffers)."""
    torch = _torch()
    return (torch.zeros if zero else torch.empty)(shape, dtype=dtype, device=device)


@dataclass
class Shard:
    rank: int
    world: int
    i0: int      # first block
    i1: int      # one past last block
    r0: int      # first permuted row
    r1: int
    p0: int      # first near pair (neighbour CSR)
    p1: int
    K0: int      # first core row
    K1: int


def shard_ranges(tess, world: int, k: int):
    """Contiguous box-row slabs, as even as possible. Returns [Shard]*world."""
    b = tess.b
    rows_of_block = tess.grid_coords[:, 0]
    slabs = int(rows_of_block.max()) + 1
    if world > slabs:
        raise ValueError(f"cannot shard {slabs} box rows over {world} ranks")
    sizes = tess.block_sizes
    ranks = np.minimum(k, sizes)
    nlen = np.array([len(x) for x in tess.neighbor_lists])
    off = np.concatenate(([0], np.cumsum(sizes)))
    roff = np.concatenate(([0], np.cumsum(ranks)))
    nptr = np.concatenate(([0], np.cumsum(nlen)))
    out = []
    for r in range(world):
        s0, s1 = (r * slabs) // world, ((r + 1) * slabs) // world
        blocks = np.flatnonzero((rows_of_block >= s0) & (rows_of_block < s1))
        i0, i1 = int(blocks[0]), int(blocks[-1]) + 1
        if i1 - i0 != len(blocks):
            raise ValueError("box-row slab is not a contiguous block range")
        out.append(Shard(r, world, i0, i1, int(off[i0]), int(off[i1]), int(nptr[i0]), int(nptr[i1]),
                         int(roff[i0]), int(roff[i1])))
    return out


@dataclass
class ShardResult:
    shard: Shard
    U: object        # (r1-r0) x k, own rows
    V: object        # N x k, all rows (gathered)
    core: object     # (K1-K0) x K, own core rows
    B: object        # own near blocks, flat, neighbour-CSR order from p0
    plan: object
    ledger: dict

    def rep_view(self, dt, k):
        """The shard's part of the compressed representation in the shape
        reconstruction.frobenius_error / frobenius_distance read: U and core
        hold this shard's rows (row0 / k0 shifts), V all rows, B this shard's
        near pairs (b0 shift)."""
        from types import SimpleNamespace
        return SimpleNamespace(dt=dt, rank=k, effective_ranks=dt.ranks(k).astype(np.int64), U=self.U, V=self.V,
                               core_d=self.core, B_d=self.B, row0=self.shard.r0, k0=self.shard.K0,
                               b0=int(dt.b_off_h[self.shard.p0]))


def torch_allgather(group=None):
    """All-gather of equal-size row shards through torch.distributed."""
    import torch.distributed as dist
    torch = _torch()

    def gather(local, total_rows):
        world = dist.get_world_size(group)
        if local.is_cuda and dist.get_backend(group) == "gloo":
            # gloo collectives run on host tensors: V is staged through host memory
            host = gather(local.cpu(), total_rows)
            return host.to(local.device)
        tail = tuple(local.shape[1:])
        sizes = torch.zeros(world, dtype=torch.int64, device=local.device)
        mine = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
        dist.all_gather_into_tensor(sizes, mine, group=group)
        sizes = [int(x) for x in sizes.cpu()]
        if sum(sizes) != total_rows:
            raise ValueError(f"shards hold {sum(sizes)} rows, expected {total_rows}")
        mx = max(sizes)
        if min(sizes) == mx:
            # every shard has total/world rows (box-row slabs of an evenly divided grid)
            out = torch.empty((total_rows,) + tail, dtype=local.dtype, device=local.device)
            dist.all_gather_into_tensor(out, local.contiguous(), group=group)
            return out
        # uneven slabs: pad every shard to the largest, gather, trim
        pad = torch.zeros((mx,) + tail, dtype=local.dtype, device=local.device)
        pad[:local.shape[0]] = local
        allp = torch.empty((world * mx,) + tail, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(allp, pad, group=group)
        return torch.cat([allp[r * mx:r * mx + s] for r, s in enumerate(sizes)], 0)

    return gather


def phase1_local(op, tess, k, p, stream, shard, plan=None, keep_sketch=False):
    """Steps 1-2 for one shard: returns (plan, U_own, V_own, dt) — the
    tagging plan, the shard's rows of U and V ((r1 - r0) x k each) and the
    device tessellation; with keep_sketch also the shard's rows of the
    sketches Y, Z ((r1 - r0) x ell (k + p), for the parity tests)."""
    torch = _torch()
    _lib.require_device()
    dt = device_tess(tess, torch.device("cuda"))
    if plan is None:
        plan = plan_tagging(tess, 0, "gaussian", stream.child(1), device=True)
    r = k + p
    gc = r
    T = plan.matrix.entries
    ell = T.shape[1]
    s = ell * gc
    G, H = draw_test_pair(dt, stream.child(0), gc)
    T_dev = _lib.h2d(T, dt.device)
    Z_dev = _lib.h2d(plan.Z, dt.device)
    _bill(op, s, s)
    inner = unwrap(op)
    if not getattr(inner, "symmetric", False) or not hasattr(inner, "device_op"):
        raise NotImplementedError("sharded compression needs a symmetric GPU kernel operator")
    nloc = shard.r1 - shard.r0
    f64 = dict(dtype=torch.float64, device=dt.device)
    Y = _alloc((nloc, s), **f64)
    Z = _alloc((nloc, s), **f64)
    st = _lib.stream_handle()
    shift = 8 * shard.r0 * s
    staged = staged_sketch_workspace(inner, dt, gc, nloc, ell)
    if staged is not None:   # A evaluated once per strip of the shard's rows, copy-only sketch producers
        _lib.call("ublr_sketch_tagged_staged", inner.device_op(dt.perm), _lib.ptr(dt.off), dt.b, _lib.ptr(T_dev), ell,
                  _lib.ptr(G), _lib.ptr(H), gc, gc, _lib.ptr(Y) - shift, _lib.ptr(Z) - shift, s, shard.r0, shard.r1,
                  0, _lib.ptr(staged[0]), staged[1], st)
        del staged
    else:
        _lib.call("ublr_sketch_tagged_pair", inner.device_op(dt.perm), _lib.ptr(dt.off), dt.b, _lib.ptr(T_dev), ell,
                  _lib.ptr(G), _lib.ptr(H), gc, gc, _lib.ptr(Y) - shift, _lib.ptr(Z) - shift, s, shard.r0, shard.r1,
                  st)
    kq = max(1, min(k, dt.m_max))
    U = _alloc((nloc, k), zero=True, **f64)
    V = _alloc((nloc, k), zero=True, **f64)
    ushift = 8 * shard.r0 * k
    _lib.call("ublr_block_qr_pair", _lib.ptr(Y) - shift, _lib.ptr(Z) - shift, s, _lib.ptr(Z_dev) + 8 * shard.i0 * ell,
              ell, gc, _lib.ptr(dt.off) + 4 * shard.i0, shard.i1 - shard.i0, kq, _lib.ptr(U) - ushift,
              _lib.ptr(V) - ushift, k, st, dt.m_max)
    if keep_sketch:
        return plan, U, V, dt, Y, Z
    del Y, Z
    return plan, U, V, dt


def phase23_local(op, k, shard, dt, U, V_all, core_out=None, panel_blocks=None):
    """Step 4: own core rows (coupling) and own near blocks (colour probes).

    The core rows land in `core_out` when given — a (K1 - K0) x K tensor on
    the device, or in PINNED HOST memory: the 1- and 2-GPU config-5 core
    (309 GB in total) does not fit in HBM, so block-row panels
    of `panel_blocks` rows are computed into two device panel buffers and
    copied out on a copy stream while the next panel is computed (the near
    field of a panel reads only that panel's core rows). A pinned `core_out`
    with FEWER rows than the shard owns is used as a ring of panel slots
    (panel n lands in slot n mod slots): the hand-off buffer of a consumer
    that drains panels as they arrive (a file writer, a sender) on a box whose
    memory cannot hold the shard's rows at all. Returns (core, B)."""
    torch = _torch()
    inner = unwrap(op)
    roff_h, roff = dt.roff(k)
    K = int(roff_h[-1])
    kloc = shard.K1 - shard.K0
    f64 = dict(dtype=torch.float64, device=dt.device)
    st = _lib.stream_handle()
    desc = inner.device_op(dt.perm)
    bbase = int(dt.b_off_h[shard.p0])
    B = _alloc((int(dt.b_off_h[shard.p1]) - bbase,), **f64)
    host = core_out is not None and not core_out.is_cuda
    if core_out is None:
        core_out = _alloc((kloc, K), **f64)
    nblk = shard.i1 - shard.i0
    pb = nblk if not host else max(1, min(nblk, panel_blocks or nblk))
    fused = dt.m_max <= FUSED_NEAR_M_MAX and min(k, dt.m_max) <= FUSED_NEAR_K_MAX and dt.pair_of is not None
    ws = None
    if not fused:
        lib = _lib.load()
        pmax = max(int(dt.nptr_h[min(a + pb, shard.i1)] - dt.nptr_h[a]) for a in range(shard.i0, shard.i1, pb))
        ws_bytes = int(lib.ublr_nearfield_workspace_bytes(pmax, max(k, 1), dt.m_max))
        ws = _alloc((max(ws_bytes, 8),), dtype=torch.uint8, device=dt.device)
    Up = _lib.ptr(U) - 8 * shard.r0 * U.stride(0)
    Bp = _lib.ptr(B) - 8 * bbase
    if host:
        rows_max = max(int(roff_h[min(a + pb, shard.i1)] - roff_h[a]) for a in range(shard.i0, shard.i1, pb))
        panels = [_alloc((rows_max, K), **f64) for _ in range(2)]
        done = [None, None]
        copy_stream = torch.cuda.Stream(device=dt.device)
        ring_slots = 0
        if core_out.shape[0] < kloc:
            ring_slots = core_out.shape[0] // rows_max
            if ring_slots < 2:
                raise ValueError(f"core_out ring needs at least {2 * rows_max} rows (two panels of {rows_max})")
    for n_, a in enumerate(range(shard.i0, shard.i1, pb)):
        e = min(a + pb, shard.i1)
        if host:
            slot = n_ % 2
            if done[slot] is not None:
                _lib.current_stream().wait_event(done[slot])     # the panel's previous copy has drained
            cbase = _lib.ptr(panels[slot]) - 8 * int(roff_h[a]) * K
        else:
            cbase = _lib.ptr(core_out) - 8 * shard.K0 * K
        if fused:
            # small blocks: core rows and near blocks from one pass over A (as direct_core)
            _lib.call("ublr_coupling_nearfield", desc, _lib.ptr(dt.off), _lib.ptr(roff), dt.b, k, Up,
                      _lib.ptr(V_all), V_all.stride(0), cbase, K, _lib.ptr(dt.cptr), _lib.ptr(dt.cidx), dt.n_colours,
                      dt.m_max, _lib.ptr(dt.pair_of), _lib.ptr(dt.nidx), _lib.ptr(dt.b_off), Bp, st, a, e)
        else:
            p0, p1 = int(dt.nptr_h[a]), int(dt.nptr_h[e])
            _lib.call("ublr_coupling", desc, _lib.ptr(dt.off), _lib.ptr(roff), dt.b, k, Up, _lib.ptr(V_all),
                      V_all.stride(0), cbase, K, st, dt.m_max, a, e)
            _lib.call("ublr_nearfield_colour", desc, _lib.ptr(dt.off), _lib.ptr(roff), dt.b, k, Up,
                      _lib.ptr(V_all), V_all.stride(0), cbase, K, _lib.ptr(dt.colours), _lib.ptr(dt.cptr),
                      _lib.ptr(dt.cidx), dt.n_colours, dt.m_max, _lib.ptr(dt.pair_i) + 4 * p0,
                      _lib.ptr(dt.nidx) + 4 * p0, p1 - p0, _lib.ptr(dt.b_off) + 8 * p0, Bp, _lib.ptr(ws),
                      ws.numel(), st)
        if host:
            r0, r1 = int(roff_h[a]) - shard.K0, int(roff_h[e]) - shard.K0
            ready = torch.cuda.Event()
            ready.record(_lib.current_stream())
            copy_stream.wait_event(ready)
            if ring_slots:
                r0, r1 = (n_ % ring_slots) * rows_max, (n_ % ring_slots) * rows_max + (r1 - r0)
            with torch.cuda.stream(copy_stream):
                core_out[r0:r1].copy_(panels[slot][:r1 - r0], non_blocking=True)
            done[slot] = torch.cuda.Event()
            done[slot].record(copy_stream)
    if host:
        _lib.current_stream().wait_stream(copy_stream)
    return core_out, B


def compress_sharded(op, tess, k, p=10, stream=None, rank=0, world=1, allgather=None, plan=None, core_out=None,
                     panel_blocks=None):
    """One rank's share of a type-A tagging (A2) compression. `core_out` /
    `panel_blocks`: see phase23_local (pinned-host core rows)."""
    stream = stream or RandomStream(0)
    cop = counting_wrapper(op)
    shard = shard_ranges(tess, world, k)[rank]
    with cop.ledger.phase("I"):
        plan, U, V, dt = phase1_local(cop, tess, k, p, stream, shard, plan)
    gather = allgather or torch_allgather()
    V_all = gather(V, dt.n)
    with cop.ledger.phase("II"):
        cop.ledger.record_apply(int(dt.roff(k)[0][-1]))
    with cop.ledger.phase("III"):
        cop.ledger.record_apply(int(sum(dt.sizes[dt.colours_h == c].max() for c in range(dt.n_colours))))
    core, B = phase23_local(op, k, shard, dt, U, V_all, core_out, panel_blocks)
    return ShardResult(shard, U, V_all, core, B, plan, cop.ledger.to_dict())


def compress_emulated(op, tess, k, p=10, stream=None, world=2):
    """All ranks of compress_sharded run one after another in this process on
    one GPU (the all-gather becomes a concatenation). Returns the list of
    ShardResults; used by the GPU tests to check sharding against the
    single-GPU pipeline."""
    torch = _torch()
    stream = stream or RandomStream(0)
    shards = shard_ranges(tess, world, k)
    plan = plan_tagging(tess, 0, "gaussian", stream.child(1), device=True)
    locs = [phase1_local(op, tess, k, p, stream, sh, plan) for sh in shards]
    V_all = torch.cat([loc[2] for loc in locs], 0)
    out = []
    for sh, (pl, U, V, dt) in zip(shards, locs):
        core, B = phase23_local(op, k, sh, dt, U, V_all)
        out.append(ShardResult(sh, U, V_all, core, B, pl, {}))
    return out
