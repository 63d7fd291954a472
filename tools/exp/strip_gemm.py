"""Strip-GEMM shapes of the staged apply (diagnostic): M x N x 65536 with the
right-hand side's own leading dimension."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2501_05528_b200 import dense as D
K = 65536
f64 = dict(dtype=torch.float64, device="cuda")
for M, N, ldb in ((7680, 4708, 4708), (7680, 4736, 4736), (7680, 4608, 4708), (4736, 4708, 4708), (1024, 4708, 4708),
                  (4736, 4096, 4096), (7680, 4708, 4712), (4096, 4708, 4708)):
    A = torch.randn(M, K, **f64)
    B = torch.randn(K, ldb, **f64)
    C = torch.zeros(M, N, **f64)
    run = lambda: D.gemm(0, 0, M, N, K, 1.0, D.addr(A), K, 0, D.addr(B), ldb, 0, 0.0, D.addr(C), N, 0, 1)
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); run(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    ct, rt = -(-N // 128), -(-M // 128)
    print(f"M{M} N{N} ldb{ldb}: {ms:8.2f} ms {2.0*M*N*K/ms/1e9:6.2f} TF/s  ctas {ct*rt} = {ct*rt/148:.2f} waves", flush=True)
    del A, B, C
