"""Check the phase-by-phase sampled CPU estimate (oracle/sampled.py) against a
full run of the oracle port on the same problem, at a size where the full
run takes minutes (diagnostic; CPU only):

    python tools/validate_sampled.py [per] [b]      (default 128 64: N = 16384, m = 256)

Prints, per method (A1 / A2 / B2 with the config-3 ranks k = 40, p = 10), the
full compression time, the sampled estimate and their ratio."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
from oracle.sampled import estimate_a1, estimate_a2, estimate_b2

per = int(sys.argv[1]) if len(sys.argv) > 1 else 128
b = int(sys.argv[2]) if len(sys.argv) > 2 else 64
k, p = 40, 10
coords = O.cell_centres(per, 2)
bx = O.partition(coords, b)
diag = -np.log(0.5 / per)
threads = os.cpu_count() or 1
op = O.KernelOp(coords, "log", diag, chunk=256, threads=threads)
for mid, est_fn in (("A1", estimate_a1), ("B2", estimate_b2), ("A2", estimate_a2)):
    t0 = time.perf_counter()
    O.compress(op, bx, k, mid, p=p, stream=O.Stream(7), compute_error=False)
    full = time.perf_counter() - t0
    est = est_fn(op, bx, k, p, label=f"N={per * per}")
    print(f"{mid} N={per * per} b={b}: full {full:.1f} s, sampled estimate {est.seconds:.1f} s "
          f"(ratio {est.seconds / full:.2f}; {est.wall:.1f} s of sampling)", flush=True)
    for row in est.table():
        print("   ", row)
