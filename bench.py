#!/usr/bin/env python
"""Benchmark: uBLR compression time on B200 (BASELINE.json metric).

    python bench.py [--config c3] [--gpus N --steps K --warmup W] [--impl reference]

One step = one full compression (phases I+II+III of
ref/reconstruction.py:498-687) of the chosen BASELINE config. Default: c3
(A1 on the 256 x 256 log-kernel grid, the largest configuration that fits one
GPU) at N = 1, and c5 (A2 on the 1024 x 1024 1/r grid, block rows sharded over
the ranks, NCCL all-gather of V) at N > 1. `--gpus N` without a torchrun
environment starts the N ranks itself.

`value` = compression time in seconds with the operator's inputs resident in
HBM (device-timed, max over ranks); `e2e` = the same through the public API
from HOST arrays (device layout and operator rebuilt from host coordinates /
matrix inside the timed region, compressed representation copied back to
pinned host memory).

Configs 1-4 do not shard: with --gpus N every rank compresses its own replica
("replicas only"). `--impl reference` times the CPU port of the
reference algorithm (oracle/, numpy + OpenBLAS on all host cores): full
compressions for c1/c2, and for c3-c5 (15-40 min on the host, or infeasible)
a phase-by-phase sampled estimate of one full compression (oracle/sampled.py),
labelled as such in the line.
"""


from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BLR compression time (s)"
FP64_PEAK_TFLOPS = 37.13  # measured DMMA m8n8k4 burst peak, profiles/fp64_peak_r01.txt
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, in-process
    through NVML (no nvidia-smi subprocess: forking one mid-region stalls the
    host thread that launches the next step); nvidia-smi only if NVML fails."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, period=0.05):
        self.index = index
        self.period = period
        self.samples = []   # (sm_mhz, max_mhz, reason bitmask)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            nv, h = self._nvml
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((float(sm), float(mx), int(rs)))
            return
        out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        if out.returncode == 0 and out.stdout.strip():
            f = [x.strip() for x in out.stdout.strip().split(",")]
            mask = sum(bit for (_, bit), v in zip(self.REASONS, f[3:7]) if v.lower().startswith("active"))
            self.samples.append((float(f[0]), float(f[1]), mask))

    def _run(self):
        while True:
            try:
                self._sample()
            except Exception:
                pass
            if self._stop.wait(self.period):
                break

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)
        try:
            self._sample()   # one sample at the end of the region
        except Exception:
            pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [x[0] for x in self.samples]
        mx = [x[1] for x in self.samples]
        reasons = sorted({name for _, _, m in self.samples for name, bit in self.REASONS if m & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def flush_l2(buf):
    buf.add_(1.0)  # 256 MB write > 126 MB L2


def free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(n):
    """`--gpus N` without a torchrun environment: start N ranks (one per GPU)
    with torch.distributed.run on this node and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def bench_config(wl, world, name, shards=None):
    """The `config` object of both arms (identical for the same workload)."""
    cfg = dict(wl.describe())
    if name == "c5":
        S = shards or world
        cfg["parallelism"] = f"block-row shards x{S}" + ("" if world == S else f" (one rank's share on {world} GPU)")
    else:
        cfg["parallelism"] = "single" if world == 1 else f"replicas x{world}"
    return cfg


def _oracle_operator(wl):
    import oracle as O
    if wl.kernel == "dense-synthetic":
        return O.Dense(wl.matrix)
    kind = "log" if wl.kernel.startswith("-log") else "inv"
    per = round(wl.n ** 0.5)
    diag = -np.log(0.5 / per) if kind == "log" else 2.0 * per
    return O.Dense(O.kernel_block(wl.points.coords, np.arange(wl.n), np.arange(wl.n), kind, diag))


def _sampled_estimate(wl):
    """oracle/sampled.py: phase-by-phase sampled timing of the oracle port at
    the full size of this workload (c3-c5)."""
    import oracle as O
    from oracle.sampled import estimate
    kind = "log" if wl.kernel.startswith("-log") else "inv"
    per = round(wl.n ** 0.5)
    diag = -np.log(0.5 / per) if kind == "log" else 2.0 * per
    bx = O.partition(wl.points.coords, wl.b)
    return estimate(wl.name, wl.points.coords, bx, wl.k, wl.p, wl.method, kind, diag)


def _cpu_line(wl, steps, warmup):
    """Times of the CPU port of the reference pipeline on this workload:
    full oracle compressions for c1/c2 (dense operator prebuilt), a sampled
    phase-by-phase estimate of one full compression for c3-c5."""
    import oracle as O
    cores = os.cpu_count() or 1
    if wl.n <= 8192:
        op = _oracle_operator(wl)
        bx = O.partition(wl.points.coords, wl.b)
        for _ in range(warmup):
            O.compress(op, bx, wl.k, wl.method, p=wl.p, stream=O.Stream(7), compute_error=False)
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            O.compress(op, bx, wl.k, wl.method, p=wl.p, stream=O.Stream(7), compute_error=False)
            times.append(time.perf_counter() - t0)
        return times, {"kind": "port", "cores": cores,
                       "sample": f"full {wl.name} compressions with the oracle numpy port (dense operator prebuilt, "
                                 f"OpenBLAS on all {cores} host threads)"}, None
    for _ in range(warmup):
        _sampled_estimate(wl)
    ests = [_sampled_estimate(wl) for _ in range(steps)]
    return [e.seconds for e in ests], {"kind": "port", "cores": cores, "sample": ests[-1].describe(),
                                       "extrapolated": True}, ests[-1].table()


def run_reference(args, rank, world, cfgname):
    """The reference arm: the CPU port of the reference pipeline (oracle/,
    numpy + OpenBLAS) on the host cores, rank 0 only."""
    if rank != 0:
        return
    from paper_2501_05528_b200 import workloads as W
    wl = W.build(cfgname, device_ops=False)
    times, info, stages = _cpu_line(wl, args.steps, args.warmup)
    v = float(np.median(times))
    line = {
        "metric": METRIC, "value": v, "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong" if cfgname == "c5" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": bench_config(wl, world, cfgname, args.shards if (cfgname == "c5" and world == 1) else None),
        "cpu_baseline": {"value": v, "unit": "s", **info},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_s": [float(t) for t in times],
    }
    if cfgname == "c5" and world == 1:
        line["value"] = line["cpu_baseline"]["value"] = line["e2e"]["value"] = v / args.shards
        line["cpu_baseline"]["sample"] += f"; divided by {args.shards} (one rank's share, as the b200 arm)"
    if stages is not None:
        line["stages"] = stages
    print(json.dumps(line))


def cpu_baseline(wl, shards=1):
    """Bounded CPU sample of the same workload with the oracle port (rank 0,
    N=1): ~12 s of full compressions for c1/c2, one sampled estimate for
    c3-c5."""
    if wl.n <= 8192:
        t_end = time.perf_counter() + 12.0
        times, info = [], None
        while time.perf_counter() < t_end or len(times) < 2:
            t, info, _ = _cpu_line(wl, 1, 0)
            times += t
        return {"value": float(np.median(times)), "unit": "s", **info,
                "sample": f"{len(times)} " + info["sample"]}
    times, info, stages = _cpu_line(wl, 1, 0)
    out = {"value": float(times[0]) / shards, "unit": "s", **info, "stages": stages}
    if shards > 1:
        out["sample"] += f"; divided by {shards} (one rank's share)"
    return out


KERNEL_OF = {"ublr_sketch_tagged_pair": "k_sketch_tagged{v} (Kronecker-restructured tagged sketch, TMEM tag groups)",
             "ublr_sketch_tagged": "k_sketch_tagged{v} (Kronecker-restructured tagged sketch, TMEM tag groups)",
             "ublr_sketch_tagged_two": "k_sketch_tagged3 (both sides of a non-symmetric A in one launch, TMEM tag groups)",
             "ublr_sketch_tagged_comp": "k_sketch_tagged4 (tagged sketch with the compensated fold, TMEM tag groups)",
             "ublr_apply": "k_apply4 (operator apply, warp-specialised: A generated by producer warps and shared by "
                           "the 2 CTAs of a cluster through st.async, DMMA consumers; the last < 512 columns on "
                           "single-CTA k_apply3 launches inside the same timed call)",
             "ublr_apply_staged": "k_gen_strip + k_gemm3 (operator apply through a staged strip of A: the strip's "
                                  "entries are evaluated once into an HBM workspace by an ALU kernel, then the "
                                  "warp-specialised stored-operand DMMA GEMM multiplies it by all w columns; the "
                                  "timed call covers every strip's two launches)",
             "ublr_gemm_batched": "k_gemm3 / k_gemm2 (batched DMMA GEMM)",
             "ublr_coupling": "k_coupling3 (C_ij = U_i^T A_ij V_j, warp-specialised)",
             "ublr_coupling_nearfield": "k_coupling_nf_small (coupling + colour-probe near field, one pass over A)"}


def kernel_label(entry, operator):
    """The kernel an entry point dispatches to for this workload (sketch.cu:
    v4 warp-specialised for the table log, v3 for 1/r and dense)."""
    return KERNEL_OF.get(entry, entry).replace("{v}", "4" if operator.startswith("-log") else "3")


def roofline_of(ev, work, config, operator):
    """Dominant C-ABI kernel by device time among those with an algorithmic
    flop count; achieved = flops / CUDA-event time of that kernel."""
    cands = [(float(np.sum(ev[k])), k) for k in ev if work.get(k, 0.0) > 0]
    if not cands:
        return None
    t_ms, name = max(cands)
    achieved = work[name] / (t_ms * 1e-3) / 1e12
    traffic = None
    tfile = os.path.join(ROOT, "profiles", f"traffic_{config}.json")
    if os.path.exists(tfile):
        tj = json.load(open(tfile))
        if tj.get("entry") == name:
            traffic = tj.get("dram_bytes_per_launch")
    n_launch = len(ev[name])
    return {"kernel": kernel_label(name, operator), "entry": name, "bound": "tensor", "pipe": "fp64 DMMA (mma.sync m8n8k4.f64)",
            "achieved": achieved,
            "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
            "peak_source": "measured DMMA m8n8k4 burst (profiles/fp64_peak_r02.txt); MEASURED_PEAKS.json has no "
                           "fp64 entry",
            "algorithmic_flops_per_launch": work[name] / n_launch, "avg_launch_ms": t_ms / n_launch,
            "launches_timed": n_launch}


def _max_over_ranks(x, world, dev):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_sharded(args, rank, world, local):
    """Config 5: block-row sharded A2. With one GPU, one rank's
    share of an --shards-way job is timed (the other shards' V rows are
    produced untimed first; the all-gather becomes a copy)."""
    import torch
    import torch.distributed as dist

    import paper_2501_05528_b200 as P
    from paper_2501_05528_b200 import _lib
    from paper_2501_05528_b200 import workloads as W
    from paper_2501_05528_b200.distributed import compress_sharded, phase1_local, shard_ranges
    from paper_2501_05528_b200.tagging import plan_tagging

    wl = W.build("c5")
    dev = torch.device("cuda", local)
    emulate = world == 1
    S = args.shards if emulate else world
    me = args.shard_rank if emulate else rank
    shards = shard_ranges(wl.tess, S, wl.k)
    other_V = None
    if emulate:   # V rows of the other shards, untimed
        stream = P.RandomStream(W.COMPRESS_SEED)
        plan0 = plan_tagging(wl.tess, 0, "gaussian", stream.child(1), device=True)
        other_V = []
        for sh in shards:
            other_V.append(None if sh.rank == me else phase1_local(wl.op, wl.tess, wl.k, wl.p, stream, sh, plan0)[2])
        torch.cuda.synchronize()

    def gather_emulated(V, n):
        return torch.cat([V if p_ is None else p_ for p_ in other_V], 0)

    # core rows of this rank: 309 GB / S. When they do not fit next to the
    # working set in HBM (S <= 2), they stream to pinned host memory in
    # block-row panels (distributed.phase23_local)
    sh = shards[me]
    K = int(np.minimum(wl.k, wl.tess.block_sizes).sum())
    core_bytes = (sh.K1 - sh.K0) * K * 8
    free, _ = torch.cuda.mem_get_info(dev)
    core_out, panel_blocks, sink = None, None, "device"
    if core_bytes > free - 24 * 2 ** 30:
        import psutil
        panel_blocks = 64
        host_free = psutil.virtual_memory().available // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
        if core_bytes > host_free - 16 * 2 ** 30:
            # neither HBM nor this rank's share of host memory holds the rows:
            # every panel is still computed and copied out, into a ring of 4
            # pinned panel slots that a file writer / sender would drain
            rows = 4 * panel_blocks * wl.k
            core_out = torch.empty((rows, K), dtype=torch.float64, pin_memory=True)
            sink = (f"pinned host RING of 4 block-row panels of 64 (rows computed and copied out, not retained: "
                    f"{core_bytes / 1e9:.0f} GB per rank fit neither in HBM nor in host memory)")
        else:
            core_out = torch.empty((sh.K1 - sh.K0, K), dtype=torch.float64, pin_memory=True)
            sink = "pinned host (block-row panels of 64)"

    def step(op=None):
        return compress_sharded(op or wl.op, wl.tess, wl.k, wl.p, P.RandomStream(W.COMPRESS_SEED), rank=me,
                                world=S, allgather=gather_emulated if emulate else None, core_out=core_out,
                                panel_blocks=panel_blocks)

    for _ in range(args.warmup):
        step()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    _lib.instrument(True)
    launches0 = _lib.launch_count
    times = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = step()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
            res = None
    ev = _lib.event_times()
    _lib.instrument(False)
    launches = (_lib.launch_count - launches0) // args.steps
    t = _max_over_ranks(float(np.mean(times)), world, dev)
    roof = roofline_of(ev, _lib.work, "c5", wl.describe().get("operator", ""))

    # e2e: operator from host coordinates (H2D), the rank's result to pinned host memory (D2H)
    e2e_times, h2d, d2h = [], 0, 0
    host = None
    for it in range(3):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        wl.tess._device.clear()
        op = P.KernelOperator(wl.points, wl.op.kind, wl.op.diag)
        h2d = wl.points.coords.nbytes
        res = step(op)
        parts = tuple(x for x in (res.U, res.core, res.B) if x.is_cuda)   # a host-sink core is already on the host
        if host is None:
            import psutil
            need = sum(x.numel() * 8 for x in parts)
            share = psutil.virtual_memory().available // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
            if need < share - 16 * 2 ** 30:
                host = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in parts]
            else:   # the rank's result does not fit in its share of host memory: through two pinned 1 GiB slots
                host = "ring"
                ring = [torch.empty(2 ** 27, dtype=torch.float64, pin_memory=True) for _ in range(2)]
                ring_ev = [None, None]
        if host == "ring":
            nslot = 0
            for x in parts:
                flat = x.reshape(-1)
                for o in range(0, flat.numel(), 2 ** 27):
                    sl = nslot % 2
                    if ring_ev[sl] is not None:
                        ring_ev[sl].synchronize()
                    chunk = flat[o:o + 2 ** 27]
                    ring[sl][:chunk.numel()].copy_(chunk, non_blocking=True)
                    ring_ev[sl] = torch.cuda.Event()
                    ring_ev[sl].record()
                    nslot += 1
        else:
            for h, x in zip(host, parts):
                h.copy_(x, non_blocking=True)
        torch.cuda.synchronize()
        d2h = sum(x.numel() * 8 for x in (res.U, res.core, res.B))
        res = parts = None
        if it > 0:
            e2e_times.append(time.perf_counter() - t0)
    e2e = _max_over_ranks(float(np.median(e2e_times)), world, dev)
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(W.build("c5", device_ops=False), shards=S)
        print(json.dumps({
            "metric": METRIC, "value": t, "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": bench_config(wl, world, "c5", S if emulate else None),
            "measured": ("one rank's share of a %d-way sharded job on 1 GPU (all-gather emulated)" % S)
            if emulate else "all ranks, NCCL all-gather of V; max over ranks",
            "shard_rank": me, "rows_per_shard": sh.r1 - sh.r0, "core_rows_in": sink,
            "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "roofline": roof,
            "kernel_ms_per_step": {k_: float(np.sum(v)) / args.steps for k_, v in ev.items()},
            "clocks": clocks.summary(), "cpu_baseline": cpu,
        }))


def run_single(args, rank, world, local, cfgname):
    import torch
    import torch.distributed as dist

    import paper_2501_05528_b200 as P
    from paper_2501_05528_b200 import _lib
    from paper_2501_05528_b200 import workloads as W

    wl = W.build(cfgname)
    dev = torch.device("cuda", local)
    l2buf = torch.zeros(32 * 1024 * 1024, dtype=torch.float64, device=dev)

    def step():
        return P.compress(wl.op, wl.tess, wl.k, wl.method, p=wl.p, stream=P.RandomStream(W.COMPRESS_SEED),
                          compute_error=False)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # one untimed instrumented step picks the dominant kernel; the timed steps
    # put CUDA events around that entry point only
    _lib.instrument(True)
    step()
    ev0 = _lib.event_times()
    cands = [(float(np.sum(v)), k) for k, v in ev0.items() if _lib.work.get(k, 0.0) > 0]
    dominant = max(cands)[1] if cands else None
    _lib.instrument(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # --- timed region: device-resident inputs -------------------------------
    _lib.instrument(True, only={dominant} if dominant else None)
    launches0 = _lib.launch_count
    step_ms = []
    gc.collect()
    small = wl.n <= 8192
    if small:
        gc.disable()   # no collector pauses inside millisecond steps
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush_l2(l2buf)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rep, report = step()
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            rep = report = None
    gc.enable()
    ev = _lib.event_times()
    _lib.instrument(False)
    launches = (_lib.launch_count - launches0) // args.steps
    t_step = _max_over_ranks(float(np.mean(step_ms)) / 1e3, world, dev)

    # --- e2e: host buffers through the public API --------------------------
    # every iteration starts from the host: a fresh device layout of the
    # tessellation, the operator from host coordinates / matrix (H2D), and
    # the compressed representation copied back to pinned host memory (D2H)
    e2e_times = []
    h2d = d2h = 0
    for it in range(max(3, args.steps // 2) + 1):   # first pass untimed (pinned staging warm-up)
        flush_l2(l2buf)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        wl.tess._device.clear()
        if wl.matrix is not None:
            op = P.DenseOperator(wl.matrix)                       # H2D of A
            h2d = wl.matrix.nbytes
        else:
            op = P.KernelOperator(wl.points, wl.op.kind, wl.op.diag)  # H2D of coordinates
            h2d = wl.points.coords.nbytes
        rep, report = P.compress(op, wl.tess, wl.k, wl.method, p=wl.p, stream=P.RandomStream(W.COMPRESS_SEED),
                                 compute_error=False)
        host = rep.to_host()                                      # D2H of the result (pinned)
        if it > 0:
            e2e_times.append(time.perf_counter() - t0)
        d2h = sum(x.nbytes for x in host.values())
        rep = report = host = None
    e2e = _max_over_ranks(float(np.median(e2e_times)), world, dev)

    roof = roofline_of(ev, _lib.work, cfgname, wl.describe().get("operator", ""))
    kernel_ms = {k: float(np.sum(v)) for k, v in ev0.items()}   # one untimed instrumented step
    if rank == 0:
        cpu = None if (args.no_cpu_baseline or world > 1) else cpu_baseline(W.build(cfgname, device_ops=False))
        line = {
            "metric": METRIC, "value": t_step, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(wl, world, cfgname),
            "timing": {"l2": "flushed between timed steps (256 MB write)",
                       "python_gc": "disabled in the timed loop" if small else "enabled (steps allocate GBs)",
                       "e2e_layout": "device tessellation layout rebuilt from host arrays every e2e step"},
            "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "roofline": roof,
            "kernel_ms_per_step": kernel_ms,
            "step_ms": {"min": float(np.min(step_ms)), "median": float(np.median(step_ms)),
                        "max": float(np.max(step_ms))},
            "phase_s": dict(P.compress(wl.op, wl.tess, wl.k, wl.method, p=wl.p,
                                       stream=P.RandomStream(W.COMPRESS_SEED), compute_error=False)[1].times_s),
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default: 30 for c1/c2, 5 for c3-c5)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None, choices=["c1", "c2", "c3", "c4", "c5"],
                    help="default: c3 (the largest single-GPU config) on 1 GPU, c5 (block-row sharded) on N > 1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shards", type=int, default=8, help="c5 on one GPU: shard count to emulate")
    ap.add_argument("--shard-rank", type=int, default=3, help="c5 on one GPU: which shard to time")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch with torchrun --nproc-per-node "
                         f"{args.gpus}, or without torchrun to let bench.py start the ranks")
    args.warmup = max(args.warmup, 3)
    cfgname = args.config or ("c3" if world == 1 else "c5")
    if args.steps is None:
        args.steps = 30 if cfgname in ("c1", "c2") else 5

    if args.impl == "reference":
        run_reference(args, rank, world, cfgname)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        if cfgname == "c5":
            run_sharded(args, rank, world, local)
        else:
            run_single(args, rank, world, local, cfgname)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
