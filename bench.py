#!/usr/bin/env python
"""Benchmark: uBLR compression time on B200 (BASELINE.json metric).

    python bench.py [--config c2] [--gpus N --steps K --warmup W] [--impl reference]

One step = one full compression (phases I+II+III of
ref/reconstruction.py:498-583: tagging plan, test-matrix generation, tagged
sketch, per-block QR, coupling, near field) of the chosen BASELINE config.
`value` = compression time in seconds with the operator's inputs resident in
HBM (device-timed, max over ranks); `e2e` = the same through the public API
from HOST arrays (operator built from host coordinates / matrix inside the
timed region, compressed representation copied back to host).

Configs 1-4 do not shard: with --gpus N every rank compresses its own replica
("replicas only"). `--impl reference` times the CPU port of the
reference algorithm (oracle/, numpy + OpenBLAS on all host cores).
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


def run_reference(args, rank, world):
    """CPU baseline: the oracle port of the reference pipeline on host cores."""
    if rank != 0:
        return
    import oracle as O
    from paper_2501_05528_b200 import workloads as W
    wl = W.build(args.config, device_ops=False)
    cores = os.cpu_count() or 1
    bx = O.partition(wl.points.coords, wl.b)
    if wl.kernel == "dense-synthetic":
        op = O.Dense(wl.matrix)
    elif wl.n <= 8192:
        kind = "log" if wl.kernel.startswith("-log") else "inv"
        diag = -np.log(0.5 / round(wl.n ** 0.5)) if kind == "log" else 2.0 * round(wl.n ** 0.5)
        op = O.Dense(O.kernel_block(wl.points.coords, np.arange(wl.n), np.arange(wl.n), kind, diag))
    else:
        raise SystemExit(json.dumps({"impl": "reference", "unavailable":
                                     f"CPU port of {args.config} exceeds the bench time budget (see DESIGN.md)"}))
    times = []
    for _ in range(args.warmup):
        O.compress(op, bx, wl.k, wl.method, p=wl.p, stream=O.Stream(7), compute_error=False)
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.compress(op, bx, wl.k, wl.method, p=wl.p, stream=O.Stream(7), compute_error=False)
        times.append(time.perf_counter() - t0)
    v = float(np.mean(times))
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {**wl.describe(), "parallelism": "cpu", "replicas": 1},
        "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "port",
                         "sample": f"full {args.config} compression (oracle/ numpy port, OpenBLAS threads={cores})"},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def cpu_baseline(wl, budget_s=12.0):
    """Bounded CPU sample of the same workload with the oracle port."""
    import oracle as O
    bx = O.partition(wl.points.coords, wl.b)
    if wl.kernel == "dense-synthetic":
        op = O.Dense(wl.matrix)
    else:
        kind = "log" if wl.kernel.startswith("-log") else "inv"
        per = round(wl.n ** 0.5)
        diag = -np.log(0.5 / per) if kind == "log" else 2.0 * per
        if wl.n > 8192:
            return None
        op = O.Dense(O.kernel_block(wl.points.coords, np.arange(wl.n), np.arange(wl.n), kind, diag))
    times = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(times) < 2:
        t0 = time.perf_counter()
        O.compress(op, bx, wl.k, wl.method, p=wl.p, stream=O.Stream(7), compute_error=False)
        times.append(time.perf_counter() - t0)
    return {"value": float(np.median(times)), "unit": "s", "cores": os.cpu_count() or 1, "kind": "port",
            "sample": f"{len(times)} full {wl.name} compressions with the oracle numpy port "
                      f"(dense operator prebuilt, OpenBLAS on all cores)"}


KERNEL_OF = {"ublr_sketch_tagged_pair": "k_sketch_tagged{v} (Kronecker-restructured tagged sketch, TMEM tag groups)",
             "ublr_sketch_tagged": "k_sketch_tagged{v} (Kronecker-restructured tagged sketch, TMEM tag groups)",
             "ublr_sketch_tagged_two": "k_sketch_tagged3 (both sides of a non-symmetric A in one launch, TMEM tag groups)",
             "ublr_apply": "k_apply3 (operator apply, warp-specialised: A generated by producer warps, DMMA consumers)",
             "ublr_gemm_batched": "k_gemm2 (batched DMMA GEMM)",
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
    return {"kernel": kernel_label(name, operator), "entry": name, "bound": "fp64", "achieved": achieved,
            "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
            "peak_source": "measured DMMA m8n8k4 burst (profiles/fp64_peak_r01.txt); MEASURED_PEAKS.json has no "
                           "fp64 entry",
            "algorithmic_flops_per_launch": work[name] / n_launch, "avg_launch_ms": t_ms / n_launch,
            "launches_timed": n_launch}


def run_sharded(args, rank, world, local):
    """Config 5: block-row sharded A2. With one GPU, one rank's
    share of an --shards-way job is timed (the other shards' V rows are
    produced untimed first; the all-gather becomes a copy)."""
    import torch
    import torch.distributed as dist

    import paper_2501_05528_b200 as P
    from paper_2501_05528_b200 import _lib
    from paper_2501_05528_b200 import workloads as W
    from paper_2501_05528_b200.distributed import (phase1_local, phase23_local, shard_ranges, torch_allgather)
    from paper_2501_05528_b200.tagging import plan_tagging

    wl = W.build(args.config)
    dev = torch.device("cuda", local)
    emulate = world == 1
    S = args.shards if emulate else world
    me = args.shard_rank if emulate else rank
    shards = shard_ranges(wl.tess, S, wl.k)
    stream = P.RandomStream(W.COMPRESS_SEED)
    other_V = None
    if emulate:   # V rows of the other shards, untimed
        plan0 = plan_tagging(wl.tess, 0, "gaussian", stream.child(1), device=True)
        parts = []
        for sh in shards:
            if sh.rank == me:
                parts.append(None)
                continue
            _, _, V, _ = phase1_local(wl.op, wl.tess, wl.k, wl.p, stream, sh, plan0)
            parts.append(V)
        other_V = parts
        torch.cuda.synchronize()

    def step():
        sh = shards[me]
        plan, U, V, dt = phase1_local(wl.op, wl.tess, wl.k, wl.p, stream, sh)
        if emulate:
            V_all = torch.cat([V if p_ is None else p_ for p_ in other_V], 0)
        else:
            V_all = torch_allgather()(V, dt.n)
        core, B = phase23_local(wl.op, wl.k, sh, dt, U, V_all)
        return core, B

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
            core, B = step()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    ev = _lib.event_times()
    _lib.instrument(False)
    launches = (_lib.launch_count - launches0) // args.steps
    t = float(np.mean(times))
    if world > 1:
        tt = torch.tensor([t], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    roof = roofline_of(ev, _lib.work, args.config, wl.describe().get("operator", ""))
    sh = shards[me]
    rows = sh.r1 - sh.r0
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": t, "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {**wl.describe(), "parallelism": f"block-row shards x{S}",
                       "measured": ("one rank's share of a %d-way sharded job on 1 GPU (all-gather emulated)" % S)
                       if emulate else "all ranks, NCCL all-gather of V",
                       "shard_rank": me, "rows_per_shard": rows},
            "gpu_launches": int(launches),
            "roofline": roof,
            "kernel_ms_per_step": {k_: float(np.sum(v)) / args.steps for k_, v in ev.items()},
            "clocks": clocks.summary(), "cpu_baseline": None,
        }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default: 30 for c1/c2, 5 for c3-c5)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shards", type=int, default=8, help="c5 on one GPU: shard count to emulate")
    ap.add_argument("--shard-rank", type=int, default=3, help="c5 on one GPU: which shard to time")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.steps is None:
        args.steps = 30 if args.config in ("c1", "c2") else 5
    rank, world, local = dist_env()

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if args.config == "c5":
        run_sharded(args, rank, world, local)
        if world > 1:
            dist.destroy_process_group()
        return

    import paper_2501_05528_b200 as P
    from paper_2501_05528_b200 import _lib
    from paper_2501_05528_b200 import workloads as W

    wl = W.build(args.config)
    flops = W.algorithmic_flops(wl)
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
    if args.config in ("c1", "c2"):
        gc.disable()   # no collector pauses inside millisecond steps (re-enabled below); c3/c4 steps
                       # allocate tens of GB, so the collector stays on there
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
    t_step = float(np.mean(step_ms)) / 1e3
    if world > 1:
        t = torch.tensor([t_step], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step = float(t.item())

    # --- e2e: host buffers through the public API --------------------------
    e2e_times = []
    h2d = d2h = 0
    host = None
    for it in range(max(3, args.steps // 2) + 1):   # first pass untimed (pinned staging warm-up)
        host = None
        flush_l2(l2buf)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
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
    e2e = float(np.median(e2e_times))
    if world > 1:
        t = torch.tensor([e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())

    # --- roofline of the dominant kernel -------------------------------------
    roof = roofline_of(ev, _lib.work, args.config, wl.describe().get("operator", ""))
    kernel_ms = {k: float(np.sum(v)) for k, v in ev0.items()}   # one untimed instrumented step

    if rank == 0:
        cpu = None if (args.no_cpu_baseline or world > 1) else cpu_baseline(W.build(args.config, device_ops=False))
        line = {
            "metric": METRIC, "value": t_step, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {**wl.describe(), "parallelism": f"replicas{world}" if world > 1 else "single",
                       "l2": "flushed between timed steps (256 MB write)", "python_gc": "disabled in the timed loop"},
            "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "roofline": roof,
            "kernel_ms_per_step": kernel_ms,
            "step_ms": {"min": float(np.min(step_ms)), "median": float(np.median(step_ms)),
                        "max": float(np.max(step_ms))},
            "phase_s": dict(report.times_s),
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
