"""Batched DMMA GEMM throughput on the shapes that dominate the c3 (A1)
block-nullification stage and the type-B solves (diagnostic):
    UBLR_GEMM_CFG=<n> python tools/gemm_bench.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2501_05528_b200 import dense as D

SHAPES = [  # (ta, tb, M, N, K, batch)
    (0, 1, 256, 256, 2354, 1433), (0, 0, 1152, 1152, 1152, 98), (0, 0, 1728, 576, 576, 98),
    (1, 0, 576, 1152, 576, 98), (1, 0, 2354, 40, 2304, 98), (0, 0, 2304, 40, 2304, 98), (1, 0, 1152, 40, 1152, 98), (0, 0, 64, 1152, 64, 98), (0, 0, 64, 40, 64, 98),
    (0, 0, 4096, 4096, 4096, 1), (1, 0, 10240, 10250, 10250, 1)]
out = []
for ta, tb, M, N, K, b in SHAPES:
    f64 = dict(dtype=torch.float64, device="cuda")
    A = torch.randn(b, (K if ta else M), (M if ta else K), **f64)
    B = torch.randn(b, (N if tb else K), (K if tb else N), **f64)
    C = torch.zeros(b, M, N, **f64)
    lda, ldb = A.shape[2], B.shape[2]
    run = lambda: D.gemm(ta, tb, M, N, K, 1.0, D.addr(A), lda, A[0].numel(), D.addr(B), ldb, B[0].numel(), 0.0,  # noqa
                         D.addr(C), N, M * N, b)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 2.0 * M * N * K * b / (ms * 1e-3) / 1e12
    print(f"cfg {os.environ.get('UBLR_GEMM_CFG', '6 (default)')} t{ta}{tb} M{M} N{N} K{K} b{b}: {ms:8.3f} ms {tf:6.2f} TF/s",
          flush=True)
    del A, B, C
