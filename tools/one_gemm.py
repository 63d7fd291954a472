"""One batched GEMM launch for ncu (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_05528_b200 import dense as D
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = torch.randn(n, n, dtype=torch.float64, device="cuda")
B = torch.randn(n, n, dtype=torch.float64, device="cuda")
C = torch.empty(n, n, dtype=torch.float64, device="cuda")
D.gemm(0, 0, n, n, n, 1.0, D.addr(A), n, 0, D.addr(B), n, 0, 0.0, D.addr(C), n, 0, 1)
torch.cuda.synchronize()
print("ok")
