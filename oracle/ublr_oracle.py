"""numpy restatement of the reference uBLR compression algorithms (oracle).

TEST INFRASTRUCTURE ONLY — see `oracle/__init__.py`. `ref/` below is
`/root/reference/pkg/src/ublr/`.

The restatement keeps the reference's index order (global point indices, not
the block-contiguous order the GPU uses), its RNG stream layout and its
numerical primitives, so that it reproduces the reference to rounding.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Stream", "philox_key", "normals", "leading_q", "null_tail", "svd_pinv",
    "power_norm", "Boxes", "cell_centres", "partition", "colour_boxes",
    "bn_width", "TagPlan", "draw_tags", "plan_tags", "b2_ok", "pair_vector",
    "Ledger", "Counted", "Bundle", "Bases", "bases_tagging", "bases_bn",
    "bases_naive", "core_direct", "near_colour_probes", "near_b2", "near_b1",
    "core_least_squares", "Compressed", "rel_error", "compress",
    "DegenerateTags",
]


# ---------------------------------------------------------------------------
# RNG — ref/linalg.py:14-52
# ---------------------------------------------------------------------------

class Stream:
    """Splittable seeded stream: numpy Philox keyed by SeedSequence(seed,
    spawn_key=key) (ref/linalg.py:22-35); normals are `standard_normal`
    filled row-major (ref/linalg.py:38-39)."""

    def __init__(self, seed, key=()):
        self.seed = int(seed)
        self.key = tuple(int(v) for v in key)
        self._g = None

    def child(self, *idx):
        return Stream(self.seed, self.key + tuple(idx))

    @property
    def gen(self):
        if self._g is None:
            ss = np.random.SeedSequence(self.seed, spawn_key=self.key)
            self._g = np.random.Generator(np.random.Philox(ss))
        return self._g

    def normal(self, rows, cols):
        return self.gen.standard_normal((rows, cols))

    def uniform(self, rows, cols):
        return self.gen.random((rows, cols))


def philox_key(seed, key=()):
    """The 128-bit Philox key numpy derives for Stream(seed, key)."""
    ss = np.random.SeedSequence(int(seed), spawn_key=tuple(int(v) for v in key))
    return ss.generate_state(2, np.uint64)


def normals(rows, cols, stream):
    """ref/linalg.py:48-52 (`gaussian`)."""
    if rows < 0 or cols < 0:
        raise ValueError("matrix dimensions must be nonnegative")
    return stream.normal(rows, cols)


# ---------------------------------------------------------------------------
# Dense kernels — ref/linalg.py:55-139
# ---------------------------------------------------------------------------

def leading_q(B, k):
    """First k columns of the unpivoted Householder Q (ref/linalg.py:55-69)."""
    B = np.asarray(B, dtype=float)
    if k > min(B.shape):
        raise ValueError(f"k={k} exceeds matrix dimensions {B.shape[0]}x{B.shape[1]}")
    if k == 0:
        return np.zeros((B.shape[0], 0))
    return np.linalg.qr(B)[0][:, :k]


def null_tail(B, k, rtol=1e-12):
    """Last k columns of the complete Q of B^T, with the reference's residual
    check (ref/linalg.py:72-94)."""
    B = np.asarray(B, dtype=float)
    ncol = B.shape[1]
    if k > ncol:
        raise ValueError(f"k={k} exceeds column count {ncol}")
    if k == 0:
        return np.zeros((ncol, 0))
    Q = np.linalg.qr(B.T, mode="complete")[0]
    Zk = Q[:, ncol - k:]
    bound = rtol * max(1.0, np.linalg.norm(B))
    res = np.linalg.norm(B @ Zk)
    if res > bound:
        raise ValueError(f"requested null space of dimension {k} does not exist "
                         f"(residual {res:.3e} > {bound:.3e})")
    return Zk


def svd_pinv(B, rtol=1e-12, with_cond=False):
    """Truncated-SVD pseudoinverse (ref/linalg.py:97-109) and, optionally, the
    untruncated condition number (ref/reconstruction.py:256-263)."""
    B = np.asarray(B, dtype=float)
    if B.size == 0:
        P = np.zeros((B.shape[1], B.shape[0]))
        return (P, np.inf) if with_cond else P
    u, s, vt = np.linalg.svd(B, full_matrices=False)
    if s[0] == 0.0:
        P = np.zeros((B.shape[1], B.shape[0]))
        return (P, np.inf) if with_cond else P
    keep = s > rtol * s[0]
    P = (vt[keep].T / s[keep]) @ u[:, keep].T
    if with_cond:
        cond = s[0] / s[-1] if s[-1] > 0 else np.inf
        return P, float(cond)
    return P


def power_norm(apply, apply_adj, n, iters=20, stream=None):
    """Power method on op*op (ref/linalg.py:112-139)."""
    if iters < 1:
        raise ValueError("iterations must be >= 1")
    stream = stream or Stream(0)
    if n == 0:
        return 0.0
    v = normals(n, 1, stream)
    nv = np.linalg.norm(v)
    if nv == 0.0:
        return 0.0
    v = v / nv
    est = 0.0
    for _ in range(iters):
        w = apply(v)
        est = float(np.linalg.norm(w))
        if est == 0.0:
            return 0.0
        v = apply_adj(w)
        v = v / np.linalg.norm(v)
    return est


# ---------------------------------------------------------------------------
# Geometry — ref/tessellation.py:44-238
# ---------------------------------------------------------------------------

def cell_centres(per_axis, d):
    """(i+0.5)/per_axis on a meshgrid(indexing='ij') (ref/tessellation.py:44-49)."""
    c = (np.arange(per_axis) + 0.5) / per_axis
    grids = np.meshgrid(*([c] * d), indexing="ij")
    return np.stack([g.ravel() for g in grids], axis=1)


@dataclass
class Boxes:
    """Box partition: `blocks[i]` ascending global indices, `nbrs[i]`
    ascending Chebyshev-1 neighbours incl. i (ref/tessellation.py:57-116)."""
    dim: int
    per_axis: int
    n: int
    blocks: list
    nbrs: list
    grid: np.ndarray
    full: bool

    @property
    def b(self):
        return len(self.blocks)

    @property
    def sizes(self):
        return np.array([len(x) for x in self.blocks])

    @property
    def m_max(self):
        return int(self.sizes.max())

    def far(self, i):
        s = set(self.nbrs[i])
        return [j for j in range(self.b) if j not in s]

    def nbr_rows(self, i):
        return np.concatenate([self.blocks[j] for j in self.nbrs[i]])

    def nbr_count(self, i):
        return int(sum(len(self.blocks[j]) for j in self.nbrs[i]))


def partition(coords, nboxes):
    """Regular grid of `nboxes` boxes; empty cells dropped
    (ref/tessellation.py:143-185)."""
    coords = np.atleast_2d(np.asarray(coords, dtype=float))
    n, d = coords.shape
    per = int(round(nboxes ** (1.0 / d)))
    per = next((c for c in (per - 1, per, per + 1) if c >= 1 and c ** d == nboxes), None)
    if per is None:
        raise ValueError(f"target_block_count={nboxes} is not a {d}-th power")
    cell = np.minimum((coords * per).astype(int), per - 1)
    flat = np.zeros(n, dtype=np.int64)
    for a in range(d):
        flat = flat * per + cell[:, a]
    order = np.argsort(flat, kind="stable")
    cut = np.flatnonzero(np.diff(flat[order])) + 1
    blocks = [np.sort(g) for g in np.split(order, cut)]
    occupied = flat[order][np.concatenate(([0], cut))]
    grid = np.zeros((len(occupied), d), dtype=int)
    rem = occupied.copy()
    for a in range(d - 1, -1, -1):
        grid[:, a] = rem % per
        rem //= per
    nbrs = []
    for i in range(len(blocks)):
        cheb = np.abs(grid - grid[i]).max(axis=1)
        nbrs.append(np.flatnonzero(cheb <= 1).tolist())
    return Boxes(d, per, n, blocks, nbrs, grid, len(blocks) == per ** d)


def colour_boxes(bx):
    """Distance-2 colouring (ref/tessellation.py:188-219): mod-3 codes on
    full grids, greedy in block order otherwise."""
    if bx.full:
        code = np.zeros(bx.b, dtype=int)
        for a in range(bx.dim):
            code = code * 3 + bx.grid[:, a] % 3
        colours = np.unique(code, return_inverse=True)[1]
    else:
        sets = [set(x) for x in bx.nbrs]
        colours = np.full(bx.b, -1, dtype=int)
        for i in range(bx.b):
            used = {colours[j] for j in range(bx.b)
                    if j != i and colours[j] >= 0 and sets[i] & sets[j]}
            c = 0
            while c in used:
                c += 1
            colours[i] = c
    return np.asarray(colours).ravel()


def bn_width(bx, r):
    """ref/bases.py:68-75."""
    return max(r + max(bx.nbr_count(i) for i in range(bx.b)), 3 ** bx.dim * r)


# ---------------------------------------------------------------------------
# Tagging planner — ref/tagging.py:23-379 (gaussian/haar, no optimisation)
# ---------------------------------------------------------------------------

class DegenerateTags(RuntimeError):
    """ref/tagging.py:23-25."""


@dataclass
class TagPlan:
    T: np.ndarray          # (b, ell)
    Z: np.ndarray          # (b, ell) per-block unit null vectors z^(i)
    rho: np.ndarray        # base aspect ratios (nan for empty far fields)
    attempts: int


def draw_tags(b, d, extra_cols, stream, distribution="gaussian"):
    """ref/tagging.py:61-91."""
    if extra_cols < 0:
        raise ValueError("extra_cols must be nonnegative")
    ell = 3 ** d + 1 + extra_cols
    if b < ell:
        raise ValueError(f"b={b} too small for {ell} tagging columns")
    if distribution == "gaussian":
        return normals(b, ell, stream)
    if distribution == "haar":
        q, r = np.linalg.qr(normals(b, ell, stream))
        sg = np.sign(np.diag(r))
        sg[sg == 0] = 1.0
        return q * sg
    raise ValueError(f"unsupported distribution {distribution!r} in the oracle")


def _plan_once(T, bx):
    """ref/tagging.py:126-139 (tag_null_vector) + :110-123 (aspect ratio) +
    :355-379 (_evaluate_plan), for optimize=False."""
    lim = 1e-12 * max(1.0, np.linalg.norm(T))
    Z = np.zeros_like(T)
    rho = np.full(bx.b, np.nan)
    for i in range(bx.b):
        sub = T[bx.nbrs[i], :]
        try:
            z = null_tail(sub, 1)[:, 0]
        except ValueError as exc:
            raise DegenerateTags(f"block {i}: {exc}") from exc
        res = float(np.linalg.norm(sub @ z))
        if res > lim:
            raise DegenerateTags(f"block {i}: null-vector residual {res:.3e}")
        Z[i] = z
        far = bx.far(i)
        if far:
            mags = np.abs((T @ z)[far])
            hi, lo = mags.max(), mags.min()
            rho[i] = 1.0 if hi == 0.0 else (np.inf if lo == 0.0 else hi / lo)
    return Z, rho


def plan_tags(bx, stream, extra_cols=0, distribution="gaussian", max_redraws=5,
              ratio_limit=1e6, extra_check=None):
    """Redraw policy of ref/tagging.py:306-352."""
    last, plan = None, None
    for attempt in range(max_redraws + 1):
        T = draw_tags(bx.b, bx.dim, extra_cols, stream.child(attempt), distribution)
        if extra_check is not None and not extra_check(T):
            last = DegenerateTags("extra_check rejected the draw")
            continue
        try:
            Z, rho = _plan_once(T, bx)
        except DegenerateTags as exc:
            last = exc
            continue
        plan = TagPlan(T, Z, rho, attempt + 1)
        fin = rho[~np.isnan(rho)]
        worst = fin.max() if fin.size else 1.0
        if np.isfinite(worst) and worst <= ratio_limit:
            return plan
    if plan is None:
        raise DegenerateTags(f"no usable tagging matrix after {max_redraws + 1} draws: {last}")
    warnings.warn(f"tagging matrix still has aspect ratio above {ratio_limit:.0e} "
                  f"after {max_redraws + 1} draws; proceeding with the last one")
    return plan


def pair_vector(T, nbrs, excluded, limit):
    """Per-pair null vector and denominator (ref/reconstruction.py:344-355)."""
    kept = [r for r in nbrs if r != excluded]
    try:
        z = null_tail(T[kept, :], 1)[:, 0]
    except ValueError as exc:
        raise DegenerateTags(str(exc)) from exc
    den = float(T[excluded] @ z)
    if abs(den) < limit:
        raise DegenerateTags(f"projected tag for pair ({nbrs}, {excluded}) vanished")
    return z, den


def b2_ok(T, bx, rtol=1e-10):
    """ref/reconstruction.py:310-323."""
    lim = rtol * max(1.0, np.linalg.norm(T))
    for i in range(bx.b):
        for j in bx.nbrs[i]:
            try:
                pair_vector(T, bx.nbrs[i], j, lim)
            except DegenerateTags:
                return False
    return True


# ---------------------------------------------------------------------------
# Ledger — ref/operators.py:75-149
# ---------------------------------------------------------------------------

class Ledger:
    def __init__(self):
        self.counts = {}
        self.phase = "other"

    def add(self, side, cols):
        self.counts.setdefault(self.phase, [0, 0])[side] += cols

    def to_dict(self):
        return {p: {"A": v[0], "Astar": v[1]} for p, v in sorted(self.counts.items())}


class Counted:
    """CountingOperator (ref/operators.py:128-149)."""

    def __init__(self, op):
        self.op = op
        self.ledger = Ledger()
        self.shape = op.shape

    def apply(self, X):
        self.ledger.add(0, X.shape[1] if X.ndim == 2 else 1)
        return self.op.apply(X)

    def apply_adjoint(self, X):
        self.ledger.add(1, X.shape[1] if X.ndim == 2 else 1)
        return self.op.apply_adjoint(X)


# ---------------------------------------------------------------------------
# Step I — ref/bases.py
# ---------------------------------------------------------------------------

@dataclass
class Bundle:
    """SketchBundle (ref/bases.py:30-46)."""
    kind: str
    omega: np.ndarray
    psi: np.ndarray
    y: np.ndarray
    z: np.ndarray
    s: int
    T: np.ndarray | None = None
    G: list | None = None
    H: list | None = None
    gc: int | None = None


@dataclass
class Bases:
    """BlockBases (ref/bases.py:49-65)."""
    U: list
    V: list
    ranks: np.ndarray
    method: str

    def offsets(self):
        return np.concatenate(([0], np.cumsum(self.ranks)))


def _basis(sample, k):
    """ref/bases.py:78-83: identity for tiny blocks, else leading Q."""
    if k >= sample.shape[0]:
        return np.eye(sample.shape[0])
    return leading_q(sample, k)


def _tagged_matrix(bx, T, blocks, gc):
    """ref/bases.py:126-137: rows of box i, group j hold t_ij * G_i."""
    out = np.zeros((bx.n, T.shape[1] * gc))
    for i, rows in enumerate(bx.blocks):
        out[rows] = np.kron(T[i], blocks[i])  # [t_i0 G_i | t_i1 G_i | ...]
    return out


def _combine(rows_y, z, gc):
    """ref/bases.py:207-210 (single null vector)."""
    m = rows_y.shape[0]
    return np.tensordot(rows_y.reshape(m, -1, gc), z, axes=(1, 0))


def bases_tagging(op, bx, k, p, plan, stream, gc=None):
    """ref/bases.py:140-204 (extra_samples=False)."""
    gc = (k + p) if gc is None else gc
    T = plan.T
    G = [normals(len(bx.blocks[i]), gc, stream.child(0, i)) for i in range(bx.b)]
    H = [normals(len(bx.blocks[i]), gc, stream.child(1, i)) for i in range(bx.b)]
    omega = _tagged_matrix(bx, T, G, gc)
    psi = _tagged_matrix(bx, T, H, gc)
    y = op.apply(omega)
    z = op.apply_adjoint(psi)
    U, V = [], []
    for i, rows in enumerate(bx.blocks):
        U.append(_basis(_combine(y[rows], plan.Z[i], gc), k))
        V.append(_basis(_combine(z[rows], plan.Z[i], gc), k))
    ranks = np.array([u.shape[1] for u in U])
    s = T.shape[1] * gc
    return Bases(U, V, ranks, "tag"), Bundle("tag", omega, psi, y, z, s, T, G, H, gc)


def bases_bn(op, bx, k, p, stream):
    """ref/bases.py:86-123."""
    r = k + p
    s = bn_width(bx, r)
    omega = normals(bx.n, s, stream.child(0))
    psi = normals(bx.n, s, stream.child(1))
    y = op.apply(omega)
    z = op.apply_adjoint(psi)
    U, V = [], []
    for i, rows in enumerate(bx.blocks):
        nr = bx.nbr_rows(i)
        U.append(_basis(y[rows] @ null_tail(omega[nr], r), k))
        V.append(_basis(z[rows] @ null_tail(psi[nr], r), k))
    ranks = np.array([u.shape[1] for u in U])
    return Bases(U, V, ranks, "bn"), Bundle("bn", omega, psi, y, z, s)


def bases_naive(op, bx, k, p, stream):
    """ref/bases.py:213-260."""
    r = k + p
    omega = np.zeros((bx.n, bx.b * r))
    psi = np.zeros((bx.n, bx.b * r))
    for i in range(bx.b):
        c = slice(i * r, (i + 1) * r)
        omega[:, c] = normals(bx.n, r, stream.child(0, i))
        psi[:, c] = normals(bx.n, r, stream.child(1, i))
        nr = bx.nbr_rows(i)
        omega[nr, c] = 0.0
        psi[nr, c] = 0.0
    y = op.apply(omega)
    z = op.apply_adjoint(psi)
    U = [_basis(y[rows, i * r:(i + 1) * r], k) for i, rows in enumerate(bx.blocks)]
    V = [_basis(z[rows, i * r:(i + 1) * r], k) for i, rows in enumerate(bx.blocks)]
    ranks = np.array([u.shape[1] for u in U])
    return Bases(U, V, ranks, "naive"), Bundle("naive", omega, psi, y, z, bx.b * r)


# ---------------------------------------------------------------------------
# Reconstruction — ref/reconstruction.py:185-421
# ---------------------------------------------------------------------------

def core_direct(op, bx, bs):
    """C = U^T (A V_blockdiag) (ref/reconstruction.py:185-198)."""
    off = bs.offsets()
    K = int(off[-1])
    Vd = np.zeros((bx.n, K))
    for j, rows in enumerate(bx.blocks):
        Vd[rows, off[j]:off[j + 1]] = bs.V[j]
    AV = op.apply(Vd)
    C = np.empty((K, K))
    for i, rows in enumerate(bx.blocks):
        C[off[i]:off[i + 1]] = bs.U[i].T @ AV[rows]
    return C


def near_colour_probes(op, bx, bs, C, colours):
    """Structured identity probes, one per colour, including the same-colour
    leak of far residuals (ref/reconstruction.py:201-244)."""
    colours = np.asarray(colours)
    for i in range(bx.b):
        nc = colours[bx.nbrs[i]]
        if len(set(nc.tolist())) != len(nc):
            raise ValueError(f"invalid coloring: two same-color probes collide in the "
                             f"neighborhood of block {i}")
    off = bs.offsets()
    sizes = bx.sizes
    B = {}
    for c in range(int(colours.max()) + 1):
        members = np.flatnonzero(colours == c)
        mc = int(sizes[members].max())
        probe = np.zeros((bx.n, mc))
        for j in members:
            probe[bx.blocks[j], :sizes[j]] = np.eye(sizes[j])
        R = op.apply(probe)
        VtP = np.empty((int(off[-1]), mc))
        for j, rows in enumerate(bx.blocks):
            VtP[off[j]:off[j + 1]] = bs.V[j].T @ probe[rows]
        CV = C @ VtP
        for i, rows in enumerate(bx.blocks):
            R[rows] -= bs.U[i] @ CV[off[i]:off[i + 1]]
        for j in members:
            for i in bx.nbrs[j]:
                B[(i, int(j))] = R[bx.blocks[i], :sizes[j]].copy()
    return B


def _perp(U, X):
    return X - U @ (U.T @ X)


def near_b1(bundle, bx, bs, cond_limit=1e8):
    """ref/reconstruction.py:266-307 (gaussian_pinv_discrepancy)."""
    left = {}
    for i, rows in enumerate(bx.blocks):
        P, cond = svd_pinv(bundle.omega[bx.nbr_rows(i)], with_cond=True)
        if cond > cond_limit:
            warnings.warn(f"block {i}: neighbor test-matrix stack has condition {cond:.2e}")
        X = _perp(bs.U[i], bundle.y[rows]) @ P
        at = 0
        for j in bx.nbrs[i]:
            w = len(bx.blocks[j])
            left[(i, j)] = X[:, at:at + w]
            at += w
    B = {}
    for j, rows in enumerate(bx.blocks):
        P, cond = svd_pinv(bundle.psi[bx.nbr_rows(j)], with_cond=True)
        if cond > cond_limit:
            warnings.warn(f"block {j}: neighbor adjoint test-matrix stack has condition {cond:.2e}")
        X = _perp(bs.V[j], bundle.z[rows]) @ P
        at = 0
        for i in bx.nbrs[j]:
            w = len(bx.blocks[i])
            Wt = X[:, at:at + w].T
            B[(i, j)] = left[(i, j)] + bs.U[i] @ (bs.U[i].T @ Wt)
            at += w
    return B


def near_b2(bundle, bx, bs, denom_rtol=1e-10):
    """ref/reconstruction.py:326-376 (tagging_pinv_discrepancy)."""
    T, gc = bundle.T, bundle.gc
    lim = denom_rtol * max(1.0, np.linalg.norm(T))
    Gp = [svd_pinv(g) for g in bundle.G]
    Hp = [svd_pinv(h) for h in bundle.H]
    left = {}
    for i, rows in enumerate(bx.blocks):
        grp = bundle.y[rows].reshape(len(rows), -1, gc)
        for j in bx.nbrs[i]:
            z, den = pair_vector(T, bx.nbrs[i], j, lim)
            left[(i, j)] = _perp(bs.U[i], np.tensordot(grp, z, axes=(1, 0))) @ Gp[j] / den
    B = {}
    for j, rows in enumerate(bx.blocks):
        grp = bundle.z[rows].reshape(len(rows), -1, gc)
        for i in bx.nbrs[j]:
            z, den = pair_vector(T, bx.nbrs[j], i, lim)
            Wt = (_perp(bs.V[j], np.tensordot(grp, z, axes=(1, 0))) @ Hp[i]).T / den
            B[(i, j)] = left[(i, j)] + bs.U[i] @ (bs.U[i].T @ Wt)
    return B


def core_least_squares(op, bundle, bx, bs, B, p, stream, max_width=None):
    """C = U^T (Y - B Omega) (V^T Omega)^+ with Gaussian augmentation
    (ref/reconstruction.py:379-421). Returns (core, extra)."""
    off = bs.offsets()
    K = int(off[-1])
    omega, y = bundle.omega, bundle.y
    extra = max(0, K + p - bundle.s)
    if extra:
        if max_width is not None and bundle.s + extra > max_width:
            raise ValueError(f"type B needs sketch width {K + p} > max_width {max_width}")
        om_x = normals(bx.n, extra, stream)
        omega = np.hstack((omega, om_x))
        y = np.hstack((y, op.apply(om_x)))
    BOm = np.zeros((bx.n, omega.shape[1]))
    for (i, j), blk in B.items():
        BOm[bx.blocks[i]] += blk @ omega[bx.blocks[j]]
    VtO = np.empty((K, omega.shape[1]))
    L = np.empty((K, omega.shape[1]))
    R = y - BOm
    for i, rows in enumerate(bx.blocks):
        VtO[off[i]:off[i + 1]] = bs.V[i].T @ omega[rows]
        L[off[i]:off[i + 1]] = bs.U[i].T @ R[rows]
    return L @ svd_pinv(VtO), extra


# ---------------------------------------------------------------------------
# Output format and pipelines — ref/reconstruction.py:50-177, :429-687
# ---------------------------------------------------------------------------

@dataclass
class Compressed:
    """UniformBLR (ref/reconstruction.py:50-132)."""
    bx: Boxes
    rank: int
    U: list
    V: list
    core: np.ndarray
    B: dict
    ranks: np.ndarray
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        near = {(i, j) for i in range(self.bx.b) for j in self.bx.nbrs[i]}
        stray = set(self.B) - near
        if stray:
            raise ValueError(f"discrepancy blocks on far-field pairs: {sorted(stray)[:4]}")

    @property
    def shape(self):
        return (self.bx.n, self.bx.n)

    def offsets(self):
        return np.concatenate(([0], np.cumsum(self.ranks)))

    def apply(self, X):
        X = np.asarray(X, dtype=float)
        off = self.offsets()
        VtX = np.empty((int(off[-1]), X.shape[1]))
        for i, rows in enumerate(self.bx.blocks):
            VtX[off[i]:off[i + 1]] = self.V[i].T @ X[rows]
        CV = self.core @ VtX
        out = np.zeros_like(X)
        for i, rows in enumerate(self.bx.blocks):
            out[rows] = self.U[i] @ CV[off[i]:off[i + 1]]
        for i, j in sorted(self.B):
            out[self.bx.blocks[i]] += self.B[(i, j)] @ X[self.bx.blocks[j]]
        return out

    def apply_adjoint(self, X):
        X = np.asarray(X, dtype=float)
        off = self.offsets()
        UtX = np.empty((int(off[-1]), X.shape[1]))
        for i, rows in enumerate(self.bx.blocks):
            UtX[off[i]:off[i + 1]] = self.U[i].T @ X[rows]
        CU = self.core.T @ UtX
        out = np.zeros_like(X)
        for i, rows in enumerate(self.bx.blocks):
            out[rows] = self.V[i] @ CU[off[i]:off[i + 1]]
        for i, j in sorted(self.B):
            out[self.bx.blocks[j]] += self.B[(i, j)].T @ X[self.bx.blocks[i]]
        return out

    def block(self, i, j):
        """Assembled block A_hat(I_i, I_j)."""
        off = self.offsets()
        out = self.U[i] @ self.core[off[i]:off[i + 1], off[j]:off[j + 1]] @ self.V[j].T
        if (i, j) in self.B:
            out = out + self.B[(i, j)]
        return out

    def to_dense(self):
        return self.apply(np.eye(self.bx.n))

    @property
    def storage_entries(self):
        return int(sum(u.size for u in self.U) + sum(v.size for v in self.V)
                   + self.core.size + sum(x.size for x in self.B.values()))


def rel_error(op, rep, iters=20, stream=None):
    """ref/reconstruction.py:160-177."""
    stream = stream or Stream(0)
    num = power_norm(lambda X: op.apply(X) - rep.apply(X),
                     lambda X: op.apply_adjoint(X) - rep.apply_adjoint(X),
                     op.shape[1], iters, stream.child(0))
    den = power_norm(op.apply, op.apply_adjoint, op.shape[1], iters, stream.child(1))
    if den == 0.0:
        raise ValueError("operator norm estimate is zero")
    return num / den


_IDS = {("A", "bn"): "A1", ("A", "tag"): "A2", ("A", "naive"): "A3",
        ("B", "bn"): "B1", ("B", "tag"): "B2"}


def compress(op, bx, k, method_id="A2", p=10, stream=None, compute_error=True,
             error_iterations=20, max_tag_redraws=5, extra_cols=0,
             distribution="gaussian", max_width=None):
    """compress / compress_type_a / compress_type_b
    (ref/reconstruction.py:498-687), optimize=False, extra_samples=False.

    Returns (Compressed, report dict with the reference's report fields)."""
    fam = {v: kk for kk, v in _IDS.items()}.get(method_id)
    if fam is None:
        raise ValueError(f"unknown method id {method_id!r}")
    family, method = fam
    stream = stream or Stream(0)
    cop = Counted(op)
    times = {}
    plan = None
    t0 = time.perf_counter()
    cop.ledger.phase = "I"
    if method == "bn":
        bs, bundle = bases_bn(cop, bx, k, p, stream.child(0))
    elif method == "naive":
        bs, bundle = bases_naive(cop, bx, k, p, stream.child(0))
    elif family == "A":
        plan = plan_tags(bx, stream.child(1), extra_cols, distribution, max_tag_redraws)
        bs, bundle = bases_tagging(cop, bx, k, p, plan, stream.child(0))
    else:
        plan = plan_tags(bx, stream.child(1), 0, distribution, max_tag_redraws,
                         extra_check=lambda T: b2_ok(T, bx))
        bs, bundle = bases_tagging(cop, bx, k, p, plan, stream.child(0), gc=bx.m_max + p)
    times["I"] = time.perf_counter() - t0
    if family == "A":
        t0 = time.perf_counter()
        cop.ledger.phase = "II"
        C = core_direct(cop, bx, bs)
        times["II"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        col = colour_boxes(bx)
        cop.ledger.phase = "III"
        B = near_colour_probes(cop, bx, bs, C, col)
        times["III"] = time.perf_counter() - t0
    else:
        t0 = time.perf_counter()
        cop.ledger.phase = "III"
        B = near_b1(bundle, bx, bs) if method == "bn" else near_b2(bundle, bx, bs)
        times["III"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        cop.ledger.phase = "II"
        C, _ = core_least_squares(cop, bundle, bx, bs, B, p, stream.child(2), max_width)
        times["II"] = time.perf_counter() - t0
    cop.ledger.phase = "other"
    rep = Compressed(bx, k, bs.U, bs.V, C, B, bs.ranks, {"method": method_id})
    rel = rel_error(op, rep, error_iterations, stream.child(9)) if compute_error else None
    report = {"method": method_id, "matvecs": cop.ledger.to_dict(), "times_s": times,
              "relative_error": rel, "storage_entries": rep.storage_entries,
              "attempts": None if plan is None else plan.attempts}
    return rep, report
