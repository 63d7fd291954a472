"""Host-side timeline of one compression (perf_counter marks only, no CUDA
events): when each pipeline function / C-ABI call starts and ends relative to
the compress() call. Diagnostic: python tools/host_timeline.py c2"""
import functools, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import _lib, bases, linalg, reconstruction, tagging, workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = W.build(cfg)
marks = []


def wrap(mod, name, label=None):
    f = getattr(mod, name)

    @functools.wraps(f)
    def g(*a, **k):
        t0 = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            marks.append((label or name, t0, time.perf_counter()))
    setattr(mod, name, g)


for mod, names in ((reconstruction, ["direct_core", "structured_identity_discrepancy", "UniformBLR", "CompressionReport",
                                     "_base_config", "_ratio_summary", "color_boxes"]),
                   (bases, ["tagging_bases", "draw_test_pair", "tagged_sketch", "block_bases_from_tagged"]),
                   (tagging, ["plan_tagging", "make_tagging_matrix", "_evaluate"]),
                   (_lib, ["h2d"])):
    for nm in names:
        wrap(mod, nm)
reconstruction.draw_test_pair = bases.draw_test_pair
if os.environ.get("TL_FINE"):
    wrap(reconstruction, "counting_wrapper")
    wrap(reconstruction, "device_tess")
    wrap(linalg, "launch_normals")
    wrap(torch, "empty", "torch.empty")
    wrap(reconstruction._PhaseTimer, "__enter__", "PhaseTimer.enter")
    wrap(reconstruction._PhaseTimer, "__exit__", "PhaseTimer.exit")
    wrap(linalg.RandomStream, "child", "RandomStream.child")
orig = _lib.call


def call(name, *a, **k):
    t0 = time.perf_counter()
    orig(name, *a, **k)
    marks.append(("C:" + name, t0, time.perf_counter()))


_lib.call = call
run = lambda: P.compress(wl.op, wl.tess, wl.k, wl.method, p=wl.p, stream=P.RandomStream(7), compute_error=False)
for _ in range(10):
    run()
torch.cuda.synchronize()
best = None
for _ in range(20):
    marks.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    if best is None or t1 - t0 < best[0]:
        best = (t1 - t0, t0, list(marks))
tot, t0, ms = best
print(f"host time of compress(): {tot * 1e3:.3f} ms")
for name, a, b in sorted(ms, key=lambda x: x[1]):
    print(f"{name:40s} {1e3 * (a - t0):8.3f} - {1e3 * (b - t0):8.3f} ms  ({1e3 * (b - a):.3f})")
