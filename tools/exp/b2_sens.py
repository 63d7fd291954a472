"""CPU experiment (oracle, N = 16384, B2): how far does A_hat move when A's
entries are perturbed at rounding level, near field only / far field only?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import oracle as O

per, nb, k, p = 128, 64, 40, 10
coords = O.cell_centres(per, 2)
bx = O.partition(coords, nb)
n = per * per
diag = -np.log(0.5 / per)
A = O.kernel_block(coords, np.arange(n), np.arange(n), "log", diag)
Afro = np.linalg.norm(A)
near = np.zeros((n, n), dtype=bool)
for i in range(nb):
    for j in bx.nbrs[i]:
        near[np.ix_(bx.blocks[i], bx.blocks[j])] = True

def run(Ap):
    t = time.time()
    rep, _ = O.compress(O.Dense(Ap), bx, k, "B2", p=p, stream=O.Stream(7), compute_error=False)
    D = rep.to_dense()
    return D, time.time() - t

D0, dt = run(A)
print(f"base: err {np.linalg.norm(A - D0) / Afro:.4e}  ({dt:.1f} s)", flush=True)
rng = np.random.default_rng(1)
for name, mask, eps in (("all 2e-16", None, 2e-16), ("far 2e-16", ~near, 2e-16), ("near 2e-16", near, 2e-16),
                        ("near 5e-14", near, 5e-14), ("all 1e-16", None, 1e-16)):
    E = rng.uniform(-1, 1, size=A.shape) * eps
    if mask is not None:
        E *= mask
    Ap = A * (1 + E)
    D, dt = run(Ap)
    print(f"{name}: ||dA||/||A|| {np.linalg.norm(Ap - A) / Afro:.2e}  ||dA_hat||/||A|| {np.linalg.norm(D - D0) / Afro:.3e}"
          f"  err vs A {np.linalg.norm(A - D) / Afro:.4e}", flush=True)
