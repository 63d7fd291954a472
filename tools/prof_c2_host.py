"""cProfile of the host side of repeated c2 compressions (diagnostic; run on
the GPU box): python tools/prof_c2_host.py [cfg] [calls]"""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
wl = W.build(cfg)


def step():
    return P.compress(wl.op, wl.tess, wl.k, wl.method, p=wl.p, stream=P.RandomStream(W.COMPRESS_SEED),
                      compute_error=False)


for _ in range(5):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    rep, report = step()
    torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(45)
st.sort_stats("cumulative").print_stats(60)
