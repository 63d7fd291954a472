"""Host cost of the primitives on a compression's critical path (diagnostic;
run on the GPU box): ctypes C-ABI calls, kernel launches, torch.empty,
torch.cuda.Event create + record."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import _lib, bases, workloads as W
from paper_2501_05528_b200.tessellation import device_tess

wl = W.build("c2")
P.compress(wl.op, wl.tess, wl.k, wl.method, p=wl.p, stream=P.RandomStream(7), compute_error=False)
torch.cuda.synchronize()
dt = device_tess(wl.tess, torch.device("cuda"))


def bench(label, fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{label:50s} {1e6 * (t1 - t0) / n:8.2f} us/call")


lib = _lib.load()
bench("ctypes ublr_last_error (no launch)", lambda: lib.ublr_last_error())
with _lib.stream_scope():
    st = P.RandomStream(7)
    tp = bases.draw_test_pair(dt, st.child(0), 30, st.child(1).child(0), 10)
    rec = dt.rng_records[next(iter(dt.rng_records))]
    buf = tp.buf
    from paper_2501_05528_b200.linalg import launch_normals
    bench("launch_normals (RNG launch via _lib.call)", lambda: launch_normals(rec, buf), 500)
    rp, cp, ns, wp, wb, _ = rec[6]
    h = _lib.stream_handle()
    fn = lib.ublr_rng_normals
    bench("raw ctypes ublr_rng_normals", lambda: fn(rp, cp, ns, buf.data_ptr(), wp, wb, h), 500)
    bench("draw_test_pair (tagged)", lambda: bases.draw_test_pair(dt, st.child(0), 30, st.child(1).child(0), 10), 500)
    bench("torch.empty 250k f64 cuda", lambda: torch.empty(250000, dtype=torch.float64, device="cuda"))
    cs = _lib.current_stream()
    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(cs)
    bench("Event(enable_timing) + record(stream)", ev)
    bench("RandomStream.child", lambda: st.child(0))
    bench("stream_scope enter/exit", lambda: _lib.stream_scope().__enter__().__exit__())
