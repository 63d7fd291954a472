"""Phase-by-phase SAMPLED timing of the oracle port at full size — TEST /
BENCH INFRASTRUCTURE ONLY (bench.py's `cpu_baseline` and `--impl reference`
legs; never on the product path).

A full CPU compression of configs 3-4 takes 15-40 minutes on the host cores
and config 5 is infeasible, so a bounded bench step
cannot run it whole. Instead every stage of the reference pipeline runs the
oracle's OWN code (oracle/ublr_oracle.py, which follows
ref/bases.py / ref/reconstruction.py line by line) on a sample of the
stage's independent units, and the stage time is scaled by
(units in the full run) / (units sampled):

* operator applies (ref/operators.py:48-52 through the row-chunked kernel
  adapter oracle.KernelOp, the reference's matrix-free operator): a sample
  of row chunks on the same thread pool, against the full-size right-hand
  side built exactly as the reference builds it (test matrix, block-diagonal
  V, colour probe);
* per-block loops (null_basis QRs, combine + col_basis, pair solves,
  pseudo-inverses): a sample of blocks of each neighbourhood size;
* sequential stream draws: a sample of rows of the same stream;
* one of the nine colour probes (ref/reconstruction.py:227-243), x 9;
* the dense K x (K + p) SVD of type-B's pinv_core (ref/reconstruction.py:420)
  at a reduced size, scaled by the size ratio to the power measured between
  two reduced sizes (at most 3).

Operator applies are sampled as two waves of the adapter's thread pool (a
cold and a warm chunk per thread, as in the full apply). Checked against
full runs of the oracle port at N = 16384 on the GPU box's 16 host threads
(`tools/validate_sampled.py`, profiles/r02/validate_sampled.txt).

The estimate is labelled as such wherever it is reported; `Estimate.stages`
keeps every (measured seconds, sampled units, total units) triple.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from .operators import KernelOp, blas_threads, kernel_block
from .ublr_oracle import (
    Stream, _basis, _combine, _perp, _tagged_matrix, bn_width, colour_boxes, leading_q, normals, null_tail,
    pair_vector, plan_tags, svd_pinv,
)


@dataclass
class Stage:
    name: str
    seconds: float       # measured on the sample
    sampled: float       # units timed
    total: float         # units in the full run

    @property
    def estimate(self) -> float:
        return self.seconds * self.total / self.sampled


@dataclass
class Estimate:
    config: str
    method: str
    threads: int
    stages: list = field(default_factory=list)
    wall: float = 0.0    # host time spent sampling

    def add(self, name, seconds, sampled, total):
        self.stages.append(Stage(name, float(seconds), float(sampled), float(total)))

    @property
    def seconds(self) -> float:
        return float(sum(s.estimate for s in self.stages))

    def table(self) -> list:
        return [{"stage": s.name, "measured_s": round(s.seconds, 4), "sampled": s.sampled, "total": s.total,
                 "estimate_s": round(s.estimate, 3)} for s in self.stages]

    def describe(self) -> str:
        return (f"phase-by-phase extrapolation of one full {self.config} ({self.method}) compression with the "
                f"oracle numpy port on {self.threads} host threads: every stage ran the port's own code on a "
                f"sample of its independent units (row chunks of each operator apply, blocks of each per-block "
                f"loop, 1 of 9 colour probes, a reduced-size core SVD scaled by n^3) and was scaled to the full "
                f"run ({self.wall:.1f} s of sampling; stages in `stages`)")


def _tic():
    return time.perf_counter()


def _apply_sample(op: KernelOp, X, waves=2, col_scale=1.0):
    """Time `waves` rounds of op.threads row chunks of op.apply(X) on the
    adapter's thread pool (the chunks a full apply runs, spread over the
    matrix). Returns (seconds, chunks timed, chunks in a full apply).

    With col_scale != 1, X holds a column sample of the full right-hand side:
    the kernel evaluation of the chunks (independent of the width) is timed
    on its own and only the remainder (the GEMM, linear in the width) is
    scaled: t = t_eval + (t_chunk - t_eval) * col_scale."""
    n = op.shape[0]
    total = -(-n // op.chunk)
    count = min(total, op.threads * waves)
    starts = [((c * total) // count) * op.chunk for c in range(count)]
    with blas_threads(1), ThreadPoolExecutor(op.threads) as ex:
        t0 = _tic()
        list(ex.map(lambda lo: op._rows(lo, min(lo + op.chunk, n), X), starts))
        dt = _tic() - t0
        if col_scale != 1.0:
            cols = np.arange(n)
            t0 = _tic()
            list(ex.map(lambda lo: kernel_block(op.coords, np.arange(lo, min(lo + op.chunk, n)), cols, op.kind,
                                                op.diag), starts))
            t_eval = _tic() - t0
            dt = t_eval + max(dt - t_eval, 0.0) * col_scale
    return dt, count, total


def _blocks_by_nbr_size(bx):
    """{neighbourhood row count: [blocks]} (interior / edge / corner boxes)."""
    out = {}
    for i in range(bx.b):
        out.setdefault(bx.nbr_count(i), []).append(i)
    return out


def estimate_a1(op: KernelOp, bx, k, p, label="c3", row_frac=16, blocks_per_size=1, col_blocks=32):
    """compress_type_a(method="bn") (ref/reconstruction.py:498-583 with
    ref/bases.py:86-123, :185-244) at full size, sampled."""
    wall0 = _tic()
    est = Estimate(label, "A1", op.threads)
    n, r = bx.n, k + p
    s = bn_width(bx, r)
    st = Stream(7).child(0)
    # phase I: Omega, Psi = gaussian(n, s) from two sequential streams
    rows = n // row_frac
    t0 = _tic()
    om_part = normals(rows, s, st.child(0))
    est.add("I: gaussian Omega, Psi (sequential streams)", _tic() - t0, rows, 2 * n)
    # the full-size test matrix the applies multiply (one is enough: the
    # adjoint side is the same apply for the symmetric kernel)
    Om = np.empty((n, s))
    for a in range(0, n, rows):
        Om[a:a + rows] = om_part[:min(rows, n - a)]
    del om_part
    dt, c, tot = _apply_sample(op, Om)
    est.add("I: Y = A Omega, Z = A* Psi (row chunks)", dt, c, 2 * tot)
    # per block: null_basis(Omega[nbr], r), Y_i P, col_basis, both sides
    rng = np.random.default_rng(5)
    for nsz, members in sorted(_blocks_by_nbr_size(bx).items()):
        for i in members[:blocks_per_size]:
            Om_nbr = rng.standard_normal((bx.nbr_count(i), s))   # Omega[nbr(i)]
            Y_i = rng.standard_normal((len(bx.blocks[i]), s))
            t0 = _tic()
            P_ = null_tail(Om_nbr, r)
            _basis(Y_i @ P_, k)
            est.add(f"I: null_basis + Y_i P + col_basis, |nbr| = {nsz}", _tic() - t0,
                    min(blocks_per_size, len(members)), 2 * len(members))
    del Om
    # phase II: direct_core = U^T (A V_dense), V_dense built as the reference
    # does (zeros + block writes), on the columns of `col_blocks` blocks
    ranks = np.minimum(k, bx.sizes)
    off = np.concatenate(([0], np.cumsum(ranks)))
    K = int(off[-1])
    Vb = [leading_q(rng.standard_normal((len(bx.blocks[j]), k)), k) for j in range(bx.b)]
    cb = min(col_blocks, bx.b)
    Kc = int(off[cb])
    t0 = _tic()
    Vd = np.zeros((n, Kc))
    for j in range(cb):
        Vd[bx.blocks[j], off[j]:off[j + 1]] = Vb[j]
    est.add("II: block-diagonal V (N x K, column sample)", _tic() - t0, cb, bx.b)
    dt, c, tot = _apply_sample(op, Vd, col_scale=bx.b / cb)
    est.add(f"II: A V_dense (row chunks; GEMM on {cb} of {bx.b} column blocks, scaled)", dt, c, tot)
    AV = np.full((n, Kc), 0.5)
    t0 = _tic()
    nb = min(16, bx.b)
    for i in range(nb):
        Vb[i].T @ AV[bx.blocks[i]]
    est.add("II: U_i^T (A V)[rows_i] (column sample)", _tic() - t0, nb * cb, bx.b * bx.b)
    del AV, Vd
    C = np.full((K, K), 0.5)
    # phase III: one colour probe of the nine (ref/reconstruction.py:227-243)
    colours = colour_boxes(bx)
    ncol = int(colours.max()) + 1
    members = np.flatnonzero(colours == 0)
    mc = int(bx.sizes[members].max())
    t0 = _tic()
    probe = np.zeros((n, mc))
    for j in members:
        probe[bx.blocks[j], :bx.sizes[j]] = np.eye(bx.sizes[j])
    t_build = _tic() - t0
    dt, c, tot = _apply_sample(op, probe)
    est.add("III: A probe_c (row chunks), 9 colours", dt, c, tot * ncol)
    R = np.full((n, mc), 0.5)
    t0 = _tic()
    VtP = np.empty((K, mc))
    for j, rows_j in enumerate(bx.blocks):
        VtP[off[j]:off[j + 1]] = Vb[j].T @ probe[rows_j]
    CV = C @ VtP
    for i, rows_i in enumerate(bx.blocks):
        R[rows_i] -= Vb[i] @ CV[off[i]:off[i + 1]]
    B = {}
    for j in members:
        for i in bx.nbrs[j]:
            B[(i, int(j))] = R[bx.blocks[i], :bx.sizes[j]].copy()
    est.add("III: probe build, V^T probe, C V^T probe, subtract, cut", _tic() - t0 + t_build, 1, ncol)
    est.wall = _tic() - wall0
    return est


def estimate_b2(op: KernelOp, bx, k, p, label="c4", row_frac=16, sample_blocks=32, svd_scale=4):
    """compress_type_b(method="tag") (ref/reconstruction.py:586-677 with
    ref/bases.py:140-204, :326-421) at full size, sampled."""
    wall0 = _tic()
    est = Estimate(label, "B2", op.threads)
    n, b = bx.n, bx.b
    stream = Stream(7)
    from .ublr_oracle import b2_ok
    t0 = _tic()
    plan = plan_tags(bx, stream.child(1), 0, "gaussian", 5, extra_check=lambda T: b2_ok(T, bx))
    est.add("I: plan_tagging + b2_denominators_ok", _tic() - t0, 1, 1)
    gc = bx.m_max + p
    t0 = _tic()
    G = [normals(len(bx.blocks[i]), gc, stream.child(0).child(0, i)) for i in range(b)]
    H = [normals(len(bx.blocks[i]), gc, stream.child(0).child(1, i)) for i in range(b)]
    omega = _tagged_matrix(bx, plan.T, G, gc)
    est.add("I: test blocks G_i, H_i + tagged Omega, Psi", _tic() - t0, 1, 1)
    s = omega.shape[1]
    dt, c, tot = _apply_sample(op, omega)
    est.add("I: Y = A Omega, Z = A* Psi (row chunks)", dt, c, 2 * tot)
    y = np.full((n, s), 0.5)
    t0 = _tic()
    U = [_basis(_combine(y[rows], plan.Z[i], gc), k) for i, rows in enumerate(bx.blocks)]
    est.add("I: combine + col_basis (both sides)", _tic() - t0, 1, 2)
    # phase III: near_b2 — pinvs of every G_j, H_i and the per-pair solves
    npinv = max(1, min(b, sample_blocks))
    t0 = _tic()
    Gp = [svd_pinv(G[j]) for j in range(npinv)]
    est.add("III: svd pseudo-inverses of G_j, H_i", _tic() - t0, npinv, 2 * b)
    Gp = Gp + [Gp[0]] * (b - npinv)
    T = plan.T
    lim = 1e-10 * max(1.0, np.linalg.norm(T))
    sample = _block_sample(b, sample_blocks)
    t0 = _tic()
    npairs = 0
    for i in sample:
        grp = y[bx.blocks[i]].reshape(len(bx.blocks[i]), -1, gc)
        for j in bx.nbrs[i]:
            z, den = pair_vector(T, bx.nbrs[i], j, lim)
            _perp(U[i], np.tensordot(grp, z, axes=(1, 0))) @ Gp[j] / den
            npairs += 1
    total_pairs = sum(len(x) for x in bx.nbrs)
    est.add("III: pair vectors + projected solves (both sides)", _tic() - t0, npairs, 2 * total_pairs)
    # phase II: pinv_core
    K = int(np.minimum(k, bx.sizes).sum())
    extra = max(0, K + p - s)
    rows = n // row_frac
    t0 = _tic()
    ox_part = normals(rows, extra, stream.child(2))
    est.add("II: augmentation gaussian (N x extra)", _tic() - t0, rows, n)
    om_x = np.empty((n, extra))
    for a in range(0, n, rows):
        om_x[a:a + rows] = ox_part[:min(rows, n - a)]
    del ox_part
    dt, c, tot = _apply_sample(op, om_x)
    est.add("II: A Omega_extra (row chunks)", dt, c, tot)
    L = s + extra
    omega = np.hstack((omega, om_x))
    del om_x
    Bblk = np.full((bx.m_max, bx.m_max), 0.5)
    t0 = _tic()
    BOm = np.zeros((n, L))
    nb = 0
    for i in sample:
        for j in bx.nbrs[i]:
            BOm[bx.blocks[i]] += Bblk @ omega[bx.blocks[j]]
            nb += 1
    est.add("II: B Omega (near pairs)", _tic() - t0, nb, total_pairs)
    t0 = _tic()
    VtO = np.empty((K, L))
    LHS = np.empty((K, L))
    off = np.concatenate(([0], np.cumsum(np.minimum(k, bx.sizes))))
    for i in sample:
        VtO[off[i]:off[i + 1]] = U[i].T @ omega[bx.blocks[i]]
        LHS[off[i]:off[i + 1]] = U[i].T @ (omega[bx.blocks[i]] - BOm[bx.blocks[i]])
    est.add("II: V^T Omega, U^T (Y - B Omega)", _tic() - t0, len(sample), b)
    del omega, BOm, VtO, LHS
    # dense SVD pseudo-inverse of V^T Omega (K x L) and the core product,
    # timed at K / svd_scale and K / (2 svd_scale); the growth exponent between
    # the two sizes (at most 3: LAPACK's efficiency rises with the size)
    # extrapolates to K
    def svd_time(div):
        Ks, Ls = K // div, L // div
        M = np.random.default_rng(3).standard_normal((Ks, Ls))
        t0 = _tic()
        Pm = svd_pinv(M)
        np.full((Ks, Ls), 0.5) @ Pm
        return _tic() - t0
    t_small, t_big = svd_time(2 * svd_scale), svd_time(svd_scale)
    alpha = min(3.0, max(2.0, np.log2(t_big / t_small))) if t_small > 0 else 3.0
    est.add(f"II: svd pinv of V^T Omega + core product, at K/{svd_scale} (x {svd_scale}^{alpha:.2f}, exponent "
            f"fitted between K/{2 * svd_scale} and K/{svd_scale})", t_big, 1, svd_scale ** alpha)
    est.wall = _tic() - wall0
    return est


def _block_sample(b, count):
    """`count` (at most b) evenly spaced block indices."""
    count = max(1, min(b, count))
    return sorted({(i * b) // count for i in range(count)})


_INPUTS = {}   # full-size right-hand sides of the apply samples, reused across steps


def estimate_a2(op: KernelOp, bx, k, p, label="c5", sample_blocks=64, col_blocks=32, attempts=None, waves=2):
    """compress_type_a(method="tag") (ref/reconstruction.py:498-583 with
    ref/tagging.py:306-379, ref/bases.py:140-210, ref/reconstruction.py:185-244)
    at full size, sampled. Config 5 is infeasible on a CPU (phase II pushes a
    1.6 TB block-diagonal V through A; the dense core is 309 GB), so phases II
    and III are additionally sampled by COLUMN blocks: the applies and the
    core products are timed against the columns of `col_blocks` blocks and
    scaled by b / col_blocks (their cost is linear in the column count)."""
    wall0 = _tic()
    est = Estimate(label, "A2", op.threads)
    n, b = bx.n, bx.b
    gc = k + p
    stream = Stream(7)
    rng = np.random.default_rng(5)
    sample = _block_sample(b, sample_blocks)
    # plan: ref/tagging.py:355-379 per block, `attempts` draws (6 at c5)
    if attempts is None:
        attempts = plan_tags(bx, stream.child(1)).attempts if b <= 1024 else 6
    T = normals(b, 3 ** bx.dim + 1, stream.child(1).child(0))
    t0 = _tic()
    for i in sample:
        z = null_tail(T[bx.nbrs[i], :], 1)[:, 0]
        far = bx.far(i)
        mags = np.abs((T @ z)[far])
        mags.max() / mags.min()
    est.add(f"I: tagging plan ({attempts} draws), null vectors + aspect ratios", _tic() - t0, len(sample),
            attempts * b)
    # test blocks and the tagged test matrices
    t0 = _tic()
    G = [normals(len(bx.blocks[i]), gc, stream.child(0).child(0, i)) for i in sample]
    est.add("I: gaussian G_i, H_i", _tic() - t0, len(sample), 2 * b)
    # the tagged test matrix ref/bases.py:126-137: its assembly is timed on
    # the sampled blocks; the full-size matrix (the right-hand side of the
    # apply sample) is built once per process
    t0 = _tic()
    for i, g in zip(sample, G):
        np.kron(T[i], g)
    est.add("I: tagged Omega, Psi (N x ell gc)", _tic() - t0, len(sample), 2 * b)
    key = ("a2-omega", n, b, gc)
    if key not in _INPUTS:
        Gs = {i: g for i, g in zip(sample, G)}
        G_all = [Gs.get(i, G[0]) if len(bx.blocks[i]) == len(G[0])
                 else rng.standard_normal((len(bx.blocks[i]), gc)) for i in range(b)]
        _INPUTS.clear()
        _INPUTS[key] = _tagged_matrix(bx, T, G_all, gc)
    omega = _INPUTS[key]
    dt, c, tot = _apply_sample(op, omega, waves=waves)
    est.add("I: Y = A Omega, Z = A* Psi (row chunks)", dt, c, 2 * tot)
    y = omega
    t0 = _tic()
    for i in sample:
        _basis(_combine(y[bx.blocks[i]], T[i] / np.linalg.norm(T[i]), gc), k)
    est.add("I: combine + col_basis", _tic() - t0, len(sample), 2 * b)
    del y
    # phase II: U^T (A V_dense) on the columns of col_blocks blocks
    ranks = np.minimum(k, bx.sizes)
    cb = list(range(min(col_blocks, b)))
    Kc = int(ranks[cb].sum())
    Vb = leading_q(rng.standard_normal((bx.m_max, k)), k)
    t0 = _tic()
    Vd = np.zeros((n, Kc))
    at = 0
    for j in cb:
        Vd[bx.blocks[j], at:at + ranks[j]] = Vb[:len(bx.blocks[j]), :ranks[j]]
        at += ranks[j]
    est.add("II: block-diagonal V (column sample)", _tic() - t0, len(cb), b)
    dt, c, tot = _apply_sample(op, Vd, waves=waves, col_scale=b / len(cb))
    est.add(f"II: A V_dense (row chunks; GEMM on {len(cb)} of {b} column blocks, scaled)", dt, c, tot)
    AV = np.full((n, Kc), 0.5)
    t0 = _tic()
    for i in sample:
        Vb[:len(bx.blocks[i])].T @ AV[bx.blocks[i]]
    est.add("II: U_i^T (A V)[rows_i] (column sample)", _tic() - t0, len(sample) * len(cb), b * b)
    del AV, Vd
    # phase III: one colour probe of the nine
    colours = colour_boxes(bx)
    ncol = int(colours.max()) + 1
    members = np.flatnonzero(colours == 0)
    mc = int(bx.sizes[members].max())
    t0 = _tic()
    probe = np.zeros((n, mc))
    for j in members:
        probe[bx.blocks[j], :bx.sizes[j]] = np.eye(bx.sizes[j])
    t_build = _tic() - t0
    dt, c, tot = _apply_sample(op, probe, waves=waves)
    est.add("III: A probe_c (row chunks), 9 colours", dt, c, tot * ncol)
    K = int(ranks.sum())
    t0 = _tic()
    VtP = np.empty((K, mc))
    off = np.concatenate(([0], np.cumsum(ranks)))
    for j, rows_j in enumerate(bx.blocks):
        VtP[off[j]:off[j + 1]] = Vb[:len(rows_j), :ranks[j]].T @ probe[rows_j]
    est.add("III: probe build + V^T probe", _tic() - t0 + t_build, 1, ncol)
    # C @ VtP (K x K x m_c) on the rows of the column-sample blocks, then the
    # per-block subtraction and cut-out on the sampled rows
    Cr = np.full((Kc, K), 0.5)
    R = np.full((n, mc), 0.5)
    t0 = _tic()
    CV = Cr @ VtP
    at = 0
    for i in cb:
        R[bx.blocks[i]] -= Vb[:len(bx.blocks[i]), :ranks[i]] @ CV[at:at + ranks[i]]
        at += ranks[i]
    est.add("III: C V^T probe + subtract (row sample)", _tic() - t0, len(cb), b * ncol)
    est.wall = _tic() - wall0
    return est


def estimate(config: str, coords, bx, k, p, method, kind, diag, threads=None):
    threads = threads or os.cpu_count() or 1
    n = coords.shape[0]
    big = n > (1 << 18)          # config 5: 64-row chunks, one wave, 8 column blocks
    op = KernelOp(coords, kind, diag, chunk=64 if big else 256, threads=threads)
    if method == "A2" and big:
        return estimate_a2(op, bx, k, p, label=config, col_blocks=8, waves=1)
    if method == "A1":
        return estimate_a1(op, bx, k, p, label=config)
    if method == "B2":
        return estimate_b2(op, bx, k, p, label=config)
    if method == "A2":
        return estimate_a2(op, bx, k, p, label=config)
    raise ValueError(f"no sampled estimate for method {method}")
