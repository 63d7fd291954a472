"""Host-submit vs GPU-execution timeline of one compression (diagnostic):
for each C-ABI launch, when the host issued it and when the GPU ran it.
python tools/timeline.py c2"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import _lib, workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = W.build(cfg)
run = lambda: P.compress(wl.op, wl.tess, wl.k, wl.method, p=wl.p, stream=P.RandomStream(7), compute_error=False)
if cfg == "c5":   # one rank's share of an 8-way job (bench.py run_sharded step)
    from paper_2501_05528_b200.distributed import phase1_local, phase23_local, shard_ranges
    sh = shard_ranges(wl.tess, 8, wl.k)[3]
    V_all = torch.zeros((wl.tess.n_points, wl.k), dtype=torch.float64, device="cuda")

    def run():
        plan, U, V, dt = phase1_local(wl.op, wl.tess, wl.k, wl.p, P.RandomStream(W.COMPRESS_SEED), sh)
        V_all[sh.r0:sh.r1] = V
        phase23_local(wl.op, wl.k, sh, dt, U, V_all)
for _ in range(2 if cfg == "c5" else 5):
    run()
torch.cuda.synchronize()
orig = _lib.call
rec = []
def call(name, *args, **kw):
    h0 = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); orig(name, *args, **kw); b.record()
    rec.append((name, h0, time.perf_counter(), a, b))
_lib.call = call
e0 = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
t0 = time.perf_counter(); e0.record()
run()
t_host = time.perf_counter() - t0
e1 = torch.cuda.Event(enable_timing=True); e1.record(); torch.cuda.synchronize()
t_end = time.perf_counter() - t0
print(f"host returns at {t_host*1e3:.3f} ms; gpu done at {e0.elapsed_time(e1):.3f} ms; wall {t_end*1e3:.3f} ms")
busy = 0.0
for name, h0, h1, a, b in rec:
    gs, ge = e0.elapsed_time(a), e0.elapsed_time(b)
    busy += ge - gs
    print(f"{name:28s} host {1e3*(h0-t0):8.3f}-{1e3*(h1-t0):8.3f}  gpu {gs:8.3f}-{ge:8.3f} ({ge-gs:.3f})")
print(f"gpu busy {busy:.3f} ms")
