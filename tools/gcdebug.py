import gc, sys, collections, time
sys.path.insert(0, '.')
import torch
import paper_2501_05528_b200 as P
from paper_2501_05528_b200 import workloads as W
wl = W.build("c2")
step = lambda: P.compress(wl.op, wl.tess, wl.k, wl.method, p=wl.p, stream=P.RandomStream(7), compute_error=False)
for _ in range(3): step()
torch.cuda.synchronize()
gc.collect()
gc.disable()
gc.set_debug(gc.DEBUG_SAVEALL)
rep, report = step()
rep = report = None
n = gc.collect()
print("collected", n)
c = collections.Counter(type(o).__name__ for o in gc.garbage)
print(c.most_common(30))
for o in gc.garbage:
    if type(o).__name__ in ("SketchBundle", "BlockBases", "UniformBLR", "TaggingPlan", "CompressionReport"):
        print(type(o).__name__, [type(r).__name__ for r in gc.get_referrers(o)][:10])
gc.set_debug(0)
gc.garbage.clear()
# time variants
import statistics
for mode in ("none", "collect", "collect0"):
    ts = []
    for _ in range(30):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = step(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        r = None
        if mode == "collect": gc.collect()
        if mode == "collect0": gc.collect(0)
    print(mode, statistics.median(ts), min(ts))
