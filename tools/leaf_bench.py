"""GPU time of the 64 x 64 leaf factorisations (diagnostic):
    UBLR_LEAF_VERSION=1|2 python tools/leaf_bench.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2501_05528_b200 import _lib
from paper_2501_05528_b200 import dense as D

b, n, nb = 98, 2304, 64
f64 = dict(dtype=torch.float64, device="cuda")
X = torch.randn(b, n, n, **f64)
G = X @ X.transpose(1, 2) / n + torch.eye(n, **f64)
R = torch.zeros_like(G)
inv = torch.zeros(b, nb, nb, **f64)
inv2 = torch.zeros_like(inv)
Dg = torch.zeros(b, n, **f64)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
W = torch.randn(b, n, n, **f64)
LU = torch.zeros_like(W)


def potrf():
    _lib.call("ublr_potrf_diag", D.addr(G), n, n * n, 0, nb, D.addr(R), n, n * n, D.addr(inv), D.addr(st), b,
              _lib.stream_handle())


def lu():
    _lib.call("ublr_lu_sign_diag_r", D.addr(W), n, n * n, 0, nb, D.addr(LU), n, n * n, D.addr(inv), D.addr(inv2),
              D.addr(Dg), n, D.addr(st), D.addr(R), n, n * n, nb, b, _lib.stream_handle())


for name, f in (("potrf_diag", potrf), ("lu_sign_diag_r", lu)):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"leaf v{os.environ.get('UBLR_LEAF_VERSION', '2')} {name}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us per launch "
          f"(batch {b}, nb {nb})")
