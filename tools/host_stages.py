"""Host-side time per pipeline function for one c2 compression (no syncs;
GPU work is asynchronous): where the Python orchestration spends its time.
python tools/host_stages.py [cfg]"""
import functools, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import _lib, bases, linalg, reconstruction, tagging, workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = W.build(cfg)
acc = {}


def wrap(mod, name):
    f = getattr(mod, name)

    @functools.wraps(f)
    def g(*a, **k):
        t0 = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            acc.setdefault(f"{mod.__name__.split('.')[-1]}.{name}", []).append(time.perf_counter() - t0)
    setattr(mod, name, g)


for mod, names in ((reconstruction, ["compress_type_a", "direct_core", "structured_identity_discrepancy",
                                     "color_boxes", "_check_coloring", "CompressionReport", "UniformBLR",
                                     "counting_wrapper", "_base_config"]),
                   (bases, ["tagging_bases", "draw_test_pair", "tagged_sketch", "block_bases_from_tagged",
                            "device_tess", "_bill"]),
                   (tagging, ["plan_tagging", "make_tagging_matrix", "_evaluate", "batched_null_vectors"]),
                   (linalg, ["device_normals_keys"]),
                   (_lib, ["call", "h2d", "stream_handle"])):
    for nm in names:
        if hasattr(mod, nm):
            wrap(mod, nm)
# modules that imported names directly
bases.device_normals_keys = linalg.device_normals_keys
run = lambda: P.compress(wl.op, wl.tess, wl.k, wl.method, p=wl.p, stream=P.RandomStream(7), compute_error=False)
for _ in range(20):
    run()
torch.cuda.synchronize()
acc.clear()
N = 50
t0 = time.perf_counter()
for _ in range(N):
    run()
    torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / N
print(f"wall per compression (synced) {tot*1e3:.3f} ms")
for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:45s} calls/run {len(v)/N:5.1f}  host ms/run {sum(v)/N*1e3:7.3f}")
