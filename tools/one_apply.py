"""One operator-apply launch for ncu (diagnostic): python tools/one_apply.py [per] [w] [kind]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_05528_b200 as P
per = int(sys.argv[1]) if len(sys.argv) > 1 else 128
w = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
kind = sys.argv[3] if len(sys.argv) > 3 else "log"
pts = P.grid_points(per, 2)
op = P.KernelOperator(pts, kind, 1.0)
perm = torch.arange(pts.n, dtype=torch.int32, device="cuda")
X = torch.randn(pts.n, w, dtype=torch.float64, device="cuda")
Y = op.apply_device(X, perm)
torch.cuda.synchronize()
print("ok", float(Y.abs().sum()))
