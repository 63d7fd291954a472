"""Compare k_apply2 tile variants (UBLR_APPLY_CFG) — diagnostic only.
python tools/apply_variants.py <variant>: prints time/TFLOPs at c3 size and
max difference against a float64 torch reference on a small problem."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2501_05528_b200 as P

def timeit(fn, reps=2):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts) / 1e3

# correctness (small): widths that take the 4-CTA cluster, 2-CTA cluster,
# single-CTA 256- and 128-column paths; n not a multiple of the 64-row tile
for per, w, kind in ((70, 700, "log"), (67, 1100, "inv"), (48, 700, "log"), (50, 1300, "log"), (50, 1300 + 512 + 100, "inv"), (37, 96, "log")):
    pts = P.grid_points(per, 2)
    n = pts.n
    op = P.KernelOperator(pts, kind, 3.0)
    perm = torch.arange(n, dtype=torch.int32, device="cuda")
    X = torch.randn(n, w, dtype=torch.float64, device="cuda")
    Y = op.apply_device(X, perm)
    c = torch.from_numpy(pts.coords).cuda()
    d2 = ((c[:, None, :] - c[None, :, :]) ** 2).sum(-1)
    A = -0.5 * torch.log(d2.fill_diagonal_(1.0)) if kind == "log" else torch.rsqrt(d2.fill_diagonal_(1.0))
    A.fill_diagonal_(3.0)
    ref = A @ X
    print("variant", os.environ.get("UBLR_APPLY_CFG", "0"), "cs", os.environ.get("UBLR_APPLY_CS", "-"), "staged", os.environ.get("UBLR_APPLY_STAGED", "1"), f"n={n} w={w} {kind}",
          "max rel diff", float((Y - ref).abs().max() / ref.abs().max()))
for kind, per, w in (("log", 256, 4096), ("log", 256, 4708), ("log", 256, 7590), ("inv", 256, 1024)):
    pts = P.grid_points(per, 2)
    n = pts.n
    op = P.KernelOperator(pts, kind, 1.0)
    perm = torch.arange(n, dtype=torch.int32, device="cuda")
    X = torch.randn(n, w, dtype=torch.float64, device="cuda")
    t = timeit(lambda: op.apply_device(X, perm), reps=1)
    fl = 2.0 * n * n * w
    print(f"  apply {kind} N={n} w={w}: {t*1e3:.1f} ms  {fl/t/1e12:.2f} TFLOP/s  ({fl/t/1e12/37.13:.1%})")
