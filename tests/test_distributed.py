"""Block-row sharding (config 5): host partition logic and the
V all-gather on CPU with gloo (world_size 2); on a GPU the emulated ranks
must reproduce the single-GPU compression exactly."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2501_05528_b200 as P
from paper_2501_05528_b200.distributed import shard_ranges, torch_allgather


@pytest.mark.parametrize("per,b,world", [(64, 64, 2), (64, 64, 4), (64, 64, 8), (48, 36, 4), (256, 256, 3)])
def test_shard_ranges_cover_everything(per, b, world):
    tess = P.build_tessellation(P.grid_points(per, 2), b)
    sh = shard_ranges(tess, world, 10)
    assert sh[0].i0 == 0 and sh[-1].i1 == tess.b
    nl = np.array([len(x) for x in tess.neighbor_lists])
    for a, c in zip(sh, sh[1:]):
        assert a.i1 == c.i0 and a.r1 == c.r0 and a.p1 == c.p0 and a.K1 == c.K0
    assert sh[-1].r1 == tess.n_points and sh[-1].p1 == nl.sum()
    # slabs are whole box rows
    rows = tess.grid_coords[:, 0]
    for s in sh:
        assert len(set(rows[s.i0:s.i1]) & set(rows[:s.i0])) == 0


def _gather_worker(rank, world, port, sizes, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    total = sum(sizes)
    full = torch.arange(total * 3, dtype=torch.float64).reshape(total, 3)
    start = sum(sizes[:rank])
    local = full[start:start + sizes[rank]].clone()
    got = torch_allgather()(local, total)
    out_q.put((rank, bool(torch.equal(got, full))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("sizes", [(4, 4), (5, 3)])
def test_allgather_gloo_world2(sizes):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + sizes[1]
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, list(sizes), q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert res == {0: True, 1: True}


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_emulated_shards_match_single_gpu(world):
    from paper_2501_05528_b200.distributed import compress_emulated
    pts = P.grid_points(64, 2)
    tess = P.build_tessellation(pts, 64)
    op = P.KernelOperator(pts, "log", -np.log(0.5 / 64))
    rep, _ = P.compress(op, tess, 20, "A2", p=10, stream=P.RandomStream(7), compute_error=False)
    parts = compress_emulated(op, tess, 20, 10, P.RandomStream(7), world=world)
    U = torch.cat([r.U for r in parts], 0)
    core = torch.cat([r.core for r in parts], 0)
    B = torch.cat([r.B for r in parts], 0)
    assert torch.equal(U, rep.U[:, :20])
    assert torch.equal(parts[0].V, rep.V[:, :20])
    assert torch.equal(core, rep.core_d)
    assert torch.equal(B, rep.B_d)


@pytest.mark.gpu
@pytest.mark.parametrize("per,b,k,kind", [(64, 64, 10, "inv"), (128, 64, 16, "inv"), (96, 36, 12, "log")])
def test_host_core_panels_match_device(per, b, k, kind):
    """Core rows streamed to pinned host memory in block-row panels (the
    1-2 GPU config-5 layout) equal the device-resident result."""
    from paper_2501_05528_b200.distributed import compress_emulated, compress_sharded
    pts = P.grid_points(per, 2)
    tess = P.build_tessellation(pts, b)
    op = P.KernelOperator(pts, kind, 2.0 * per if kind == "inv" else -np.log(0.5 / per))
    world = 2
    ref = compress_emulated(op, tess, k, 8, P.RandomStream(3), world=world)
    V_all = ref[0].V
    for r in range(world):
        sh = ref[r].shard
        host = torch.empty(ref[r].core.shape, dtype=torch.float64, pin_memory=True)
        res = compress_sharded(op, tess, k, 8, P.RandomStream(3), rank=r, world=world,
                               allgather=lambda V, n: V_all, core_out=host, panel_blocks=3)
        torch.cuda.synchronize()
        assert res.core is host
        assert torch.equal(host, ref[r].core.cpu())
        assert torch.equal(res.B, ref[r].B)
        assert res.shard == sh


@pytest.mark.gpu
def test_host_core_ring_holds_last_panels():
    """A pinned core_out with fewer rows than the shard owns is a ring of
    panel slots: after the run, slot (n mod slots) holds panel n for the last
    panels; near blocks are unaffected."""
    from paper_2501_05528_b200.distributed import compress_emulated, compress_sharded
    per, b, k, pb = 48, 36, 8, 2
    pts = P.grid_points(per, 2)
    tess = P.build_tessellation(pts, b)
    op = P.KernelOperator(pts, "log", -np.log(0.5 / per))
    ref = compress_emulated(op, tess, k, 8, P.RandomStream(3), world=1)[0]
    rows_max = pb * k
    slots = 3
    ring = torch.zeros((slots * rows_max, ref.core.shape[1]), dtype=torch.float64, pin_memory=True)
    res = compress_sharded(op, tess, k, 8, P.RandomStream(3), rank=0, world=1, allgather=lambda V, n: V,
                           core_out=ring, panel_blocks=pb)
    torch.cuda.synchronize()
    assert torch.equal(res.B, ref.B)
    npan = b // pb
    core = ref.core.cpu()
    for n in range(npan - slots, npan):
        want = core[n * rows_max:(n + 1) * rows_max]
        got = ring[(n % slots) * rows_max:(n % slots + 1) * rows_max]
        assert torch.equal(got, want)


def _sharded_worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2501_05528_b200.distributed import compress_sharded
    pts = P.grid_points(64, 2)
    tess = P.build_tessellation(pts, 64)
    op = P.KernelOperator(pts, "inv", 128.0)
    res = compress_sharded(op, tess, 10, 6, P.RandomStream(11), rank=rank, world=world)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), U=res.U.cpu().numpy(), V=res.V.cpu().numpy(),
             core=res.core.cpu().numpy(), B=res.B.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_multiprocess_sharded_gloo_matches_emulated(tmp_path):
    """Two ranks as two processes (gloo; V staged through host memory — the
    NCCL path of bench.py on an 8-GPU box), each computing its shard on the
    device, against the in-process emulation of the same ranks."""
    from paper_2501_05528_b200.distributed import compress_emulated
    ctx = mp.get_context("spawn")
    port = 29700 + (os.getpid() % 500)
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, str(tmp_path))) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    pts = P.grid_points(64, 2)
    tess = P.build_tessellation(pts, 64)
    ref = compress_emulated(P.KernelOperator(pts, "inv", 128.0), tess, 10, 6, P.RandomStream(11), world=2)
    for r in range(2):
        got = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(got["U"], ref[r].U.cpu().numpy())
        assert np.array_equal(got["V"], ref[r].V.cpu().numpy())
        assert np.array_equal(got["core"], ref[r].core.cpu().numpy())
        assert np.array_equal(got["B"], ref[r].B.cpu().numpy())


class _GuardedAlloc:
    """Every buffer is the middle of a larger one whose two guard bands hold a
    sentinel bit pattern; `check()` verifies no kernel wrote outside its
    buffer (compute-sanitizer is unavailable on this pool, so out-of-bounds
    writes of the shifted shard pointers are caught this way)."""

    GUARD = 1 << 16   # elements per side

    def __init__(self):
        self.blocks = []

    def __call__(self, shape, dtype=None, device=None, zero=False):
        n = int(np.prod(shape))
        big = torch.empty(n + 2 * self.GUARD, dtype=dtype, device=device)
        raw = big.view(torch.uint8)
        raw.fill_(0xA5)
        body = big[self.GUARD:self.GUARD + n]
        if zero:
            body.zero_()
        self.blocks.append(big)
        return body.view(shape)

    def check(self):
        torch.cuda.synchronize()
        for big in self.blocks:
            raw = big.view(torch.uint8)
            g = self.GUARD * big.element_size()
            assert bool((raw[:g] == 0xA5).all()) and bool((raw[-g:] == 0xA5).all()), "write outside a buffer"


@pytest.mark.gpu
@pytest.mark.parametrize("per,b,k,world,kind", [(256, 256, 48, 8, "inv"), (64, 64, 10, 4, "inv"),
                                                (96, 36, 12, 3, "log")])
def test_shard_kernels_stay_inside_their_buffers(monkeypatch, per, b, k, world, kind):
    """Guard bands around every shard buffer (Y, Z, U, V, core rows, near
    blocks, workspace, host-sink panels) for each rank of a sharded job,
    with the result compared against the unguarded run."""
    import paper_2501_05528_b200.distributed as Dm
    pts = P.grid_points(per, 2)
    tess = P.build_tessellation(pts, b)
    op = P.KernelOperator(pts, kind, 2.0 * per if kind == "inv" else -np.log(0.5 / per))
    ref = Dm.compress_emulated(op, tess, k, 16, P.RandomStream(5), world=world)
    guard = _GuardedAlloc()
    monkeypatch.setattr(Dm, "_alloc", guard)
    got = Dm.compress_emulated(op, tess, k, 16, P.RandomStream(5), world=world)
    host = torch.empty(got[1].core.shape, dtype=torch.float64, pin_memory=True)
    V_all = got[0].V
    panel = Dm.compress_sharded(op, tess, k, 16, P.RandomStream(5), rank=1, world=world,
                                allgather=lambda V, n: V_all, core_out=host, panel_blocks=2)
    guard.check()
    for a, c in zip(ref, got):
        assert torch.equal(a.core, c.core) and torch.equal(a.B, c.B) and torch.equal(a.U, c.U)
    assert torch.equal(host, ref[1].core.cpu())
    assert len(guard.blocks) >= 6 * world
