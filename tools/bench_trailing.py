"""Microbenchmark: batched trailing updates C -= A B (the blocked LU/Cholesky
shapes of the c3 block-nullification stage), CUDA-event timed.
python tools/bench_trailing.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_05528_b200 import dense as D, _lib

def t_ms(f, reps=5):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

batch, n = 98, 2304
C = torch.randn(batch, n, n, dtype=torch.float64, device="cuda")
for n2 in (2240, 1600, 960):
    for K in (64, 128):
        A = torch.randn(batch, n2, K, dtype=torch.float64, device="cuda")
        B = torch.randn(batch, K, n2, dtype=torch.float64, device="cuda")
        f = lambda: D.gemm(0, 0, n2, n2, K, -1.0, D.addr(A), K, n2 * K, D.addr(B), n2, n2 * K, 1.0,
                           D.addr(C, n - n2), n, n * n, batch)
        ms = t_ms(f)
        fl = 2.0 * n2 * n2 * K * batch
        g = lambda: _lib.call("ublr_syrk_upper_batched", n2, K, -1.0, D.addr(B), n2, n2 * K, 1.0, D.addr(C, n - n2),
                              n, n * n, batch, _lib.stream_handle())
        ms2 = t_ms(g)
        print(f"n2={n2} K={K}: gemm {ms:.3f} ms {fl / ms / 1e9:.1f} TF/s | syrk {ms2:.3f} ms "
              f"{fl / 2 / ms2 / 1e9:.1f} TF/s(alg)")
