"""Kernel microbenchmarks on the GPU (CUDA-event timed): operator apply,
batched GEMM, tagged sketch. Usage: python tools/kbench.py [apply|gemm|sketch ...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import _lib, dense as D
from paper_2501_05528_b200.tessellation import device_tess

def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts) / 1e3

def bench_apply():
    for kind, per, w in (("log", 181, 1024), ("inv", 181, 1024), ("log", 256, 4708)):
        pts = P.grid_points(per, 2)
        n = pts.n
        op = P.KernelOperator(pts, kind, 1.0)
        perm = torch.arange(n, dtype=torch.int32, device="cuda")
        X = torch.randn(n, w, dtype=torch.float64, device="cuda")
        t = timeit(lambda: op.apply_device(X, perm), reps=2)
        fl = 2.0 * n * n * w
        print(f"apply {kind} N={n} w={w}: {t*1e3:.1f} ms  {fl/t/1e12:.2f} TFLOP/s  ({fl/t/1e12/37.13:.1%} of 37.1)")

def bench_gemm():
    for (b, M, N, K, ta, tb) in ((64, 2304, 2304, 2354, 0, 1), (1, 8192, 8192, 8192, 0, 0), (256, 256, 10250, 256, 0, 0)):
        A = torch.randn(b, M, K, dtype=torch.float64, device="cuda") if not ta else torch.randn(b, K, M, dtype=torch.float64, device="cuda")
        B = torch.randn(b, K, N, dtype=torch.float64, device="cuda") if not tb else torch.randn(b, N, K, dtype=torch.float64, device="cuda")
        C = torch.empty(b, M, N, dtype=torch.float64, device="cuda")
        lda = A.shape[2]; ldb = B.shape[2]
        f = lambda: D.gemm(ta, tb, M, N, K, 1.0, D.addr(A), lda, A.shape[1] * A.shape[2], D.addr(B), ldb,
                           B.shape[1] * B.shape[2], 0.0, D.addr(C), N, M * N, b)
        t = timeit(f)
        fl = 2.0 * b * M * N * K
        ref = torch.matmul(A if not ta else A.transpose(1, 2), B if not tb else B.transpose(1, 2))
        err = (ref - C).abs().max().item() / ref.abs().max().item()
        print(f"gemm b={b} {M}x{N}x{K} ta={ta} tb={tb}: {t*1e3:.1f} ms {fl/t/1e12:.2f} TFLOP/s ({fl/t/1e12/37.13:.1%}) err {err:.1e}")

def bench_sketch():
    from paper_2501_05528_b200.bases import draw_test_blocks, tagged_sketch
    for per, b, gc, kind in ((64, 64, 30, "log"), (256, 256, 64, "inv"), (256, 256, 266, "log")):
        pts = P.grid_points(per, 2)
        tess = P.build_tessellation(pts, b)
        dt = device_tess(tess, torch.device("cuda"))
        op = P.KernelOperator(pts, kind, 1.0)
        plan = P.plan_tagging(tess, 0, "gaussian", P.RandomStream(7).child(1))
        G = draw_test_blocks(dt, P.RandomStream(1), 0, gc)
        H = draw_test_blocks(dt, P.RandomStream(1), 1, gc)
        T = torch.from_numpy(plan.matrix.entries).cuda()
        t = timeit(lambda: tagged_sketch(op, dt, T, plan.matrix.entries, G, H, gc), reps=2)
        n = pts.n
        fl = 2 * (2.0 * n * n * gc + 2.0 * n * b * gc * 10)
        print(f"sketch {kind} N={n} b={b} gc={gc}: {t*1e3:.2f} ms {fl/t/1e12:.2f} TFLOP/s ({fl/t/1e12/37.13:.1%})")

def bench_coupling():
    from paper_2501_05528_b200.bases import BlockBases
    from paper_2501_05528_b200.reconstruction import direct_core
    for per, b, k, kind in ((256, 256, 48, "inv"), (256, 256, 40, "log"), (64, 64, 20, "log")):
        pts = P.grid_points(per, 2)
        tess = P.build_tessellation(pts, b)
        dt = device_tess(tess, torch.device("cuda"))
        op = P.KernelOperator(pts, kind, 1.0)
        U = torch.randn(dt.n, k, dtype=torch.float64, device="cuda")
        bs = BlockBases(dt, U, U.clone(), k, "tag", (0, 0))
        t = timeit(lambda: direct_core(op, tess, bs), reps=2)
        n = dt.n
        fl = 2.0 * n * n * k + 2.0 * n * (b * k) * k
        print(f"coupling {kind} N={n} b={b} k={k}: {t*1e3:.2f} ms {fl/t/1e12:.2f} TFLOP/s ({fl/t/1e12/37.13:.1%})")


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for what in (sys.argv[1:] or ["apply", "gemm", "sketch", "coupling"]):
        globals()["bench_" + what]()

