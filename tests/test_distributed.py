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
