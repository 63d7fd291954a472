"""Tagging planner (host side; ref/tagging.py:23-379).

The b x ell tagging matrix T, the per-block null vectors z^(i) of T(N_i, :)
and the per-pair vectors of T(N_i \\ {j}, :) are tiny host problems, but their
exact values matter (boundary blocks have nullity >= 2, so a different
orthonormalisation changes the sample: SURVEY.md F2, F13). They are computed
with numpy's own Householder QR, exactly as the reference does, but batched:
all blocks with the same neighbour count go through one stacked
`np.linalg.qr` call (the reference loops in Python, which costs 10 s of
phase I at b = 4096).
"""

from __future__ import annotations

import warnings
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np

from .linalg import RandomStream, gaussian
from .tessellation import Tessellation


class DegenerateTagsError(RuntimeError):
    """ref/tagging.py:23-25."""


@dataclass(frozen=True)
class TaggingMatrix:
    entries: np.ndarray
    dim: int
    extra_cols: int
    distribution: str
    seed: int

    @property
    def b(self) -> int:
        return self.entries.shape[0]

    @property
    def n_cols(self) -> int:
        return self.entries.shape[1]


@dataclass(frozen=True)
class NullVector:
    block: int
    vector: np.ndarray
    residual: float


@dataclass(frozen=True)
class ProjectedTags:
    block: int
    values: np.ndarray


class NullVectors(Sequence):
    """The per-block NullVector records of a plan, materialised on access
    (the plan keeps the stacked (b, ell) array)."""

    def __init__(self, Z, res):
        self.Z, self.res = Z, res

    def __len__(self):
        return self.Z.shape[0]

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        return NullVector(block=int(i), vector=self.Z[i], residual=float(self.res[i]))


@dataclass
class TaggingPlan:
    matrix: TaggingMatrix
    null_vectors: list
    rho_base: np.ndarray
    rho_optimized: np.ndarray | None
    attempts: int

    @property
    def Z(self) -> np.ndarray:
        """(b, ell) stacked null vectors."""
        if isinstance(self.null_vectors, NullVectors):
            return self.null_vectors.Z
        return np.stack([nv.vector for nv in self.null_vectors])


DISTRIBUTIONS = ("gaussian", "haar", "equidistributed")


def make_tagging_matrix(b, d, extra_cols=0, distribution="gaussian", stream=None) -> TaggingMatrix:
    """ref/tagging.py:61-91 (gaussian and haar)."""
    stream = stream or RandomStream(0)
    if extra_cols < 0:
        raise ValueError("extra_cols must be nonnegative")
    ell = 3 ** d + 1 + extra_cols
    if b < ell:
        raise ValueError(f"b={b} too small for {ell} tagging columns")
    if distribution == "gaussian":
        entries = gaussian(b, ell, stream)
    elif distribution == "haar":
        q, r = np.linalg.qr(gaussian(b, ell, stream))
        signs = np.sign(np.diag(r))
        signs[signs == 0] = 1.0
        entries = q * signs
    elif distribution == "equidistributed":
        entries = equidistributed_rows(b, ell, stream)
    else:
        raise ValueError(f"unknown distribution {distribution!r}; expected one of {DISTRIBUTIONS}")
    return TaggingMatrix(entries, d, extra_cols, distribution, stream.seed)


def equidistributed_rows(b, ell, stream, iterations=200):
    """ref/tagging.py:94-123: normalised Gaussian rows spread over the unit
    sphere by Riesz-energy descent against the other rows and their antipodes
    (step 0.25 d_min^3, displacement capped at d_min / 2, renormalised after
    each step). Host planning: b x b x ell work per iteration, done once per
    draw before any kernel runs."""
    rows = gaussian(b, ell, stream)
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    for _ in range(iterations):
        force = np.zeros_like(rows)
        d_min = np.inf
        for sgn in (1.0, -1.0):
            diff = rows[:, None, :] - sgn * rows[None, :, :]
            d2 = (diff ** 2).sum(axis=2)
            d2[d2 < 1e-30] = np.inf
            dist = np.sqrt(d2)
            force += (diff / dist[:, :, None] ** 3).sum(axis=1)
            d_min = min(d_min, dist.min())
        disp = (0.25 * d_min ** 3) * force
        dlen = np.linalg.norm(disp, axis=1, keepdims=True)
        rows = rows + disp * np.minimum(1.0, (0.5 * d_min) / np.maximum(dlen, 1e-300))
        rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    return rows


def _csr(rows_list):
    ptr = np.zeros(len(rows_list) + 1, dtype=np.int32)
    ptr[1:] = np.cumsum([len(r) for r in rows_list])
    idx = np.concatenate([np.asarray(r, dtype=np.int32) for r in rows_list]) if rows_list else np.zeros(0, np.int32)
    return ptr, np.ascontiguousarray(idx, dtype=np.int32)


def _fro(E) -> float:
    """||E||_F. np.linalg.norm of a 2-D array goes through a BLAS dot that
    cost 30+ ms for a 4096 x 10 tagging matrix on the bench hosts (thread
    start-up); the residual limits only need the value to rounding."""
    E = np.asarray(E, dtype=np.float64)
    return float(np.sqrt(np.einsum("ij,ij->", E, E)))


def _neighbour_csr(tess):
    """CSR of the neighbour lists, cached on the tessellation."""
    c = tess._device.get("nbr_csr")
    if c is None:
        c = _csr(tess.neighbor_lists)
        tess._device["nbr_csr"] = c
    return c


def batched_null_vectors(T: np.ndarray, rows_list: list, rtol: float = 1e-12, csr=None):
    """Last column of the complete QR of T[rows]^T for every row set
    (== null_basis(T[rows], 1)[:, 0], ref/linalg.py:72-94), by the C-ABI host
    function ublr_null_vectors (Householder in LAPACK's convention; equal to
    numpy's qr(mode="complete") up to rounding, checked in tests/test_host.py).

    Returns (Z (n_sets, ell), residual ||T[rows] z|| (n_sets,), ok mask where
    the reference's residual test passes)."""
    from . import _lib

    T = np.ascontiguousarray(T, dtype=np.float64)
    ell = T.shape[1]
    ptr, idx = csr if csr is not None else _csr(rows_list)
    n = len(ptr) - 1
    if n and int(np.diff(ptr).max()) >= ell:
        raise DegenerateTagsError("requested null space of dimension 1 does not exist")
    Z = np.zeros((n, ell))
    res = np.zeros(n)
    _lib.check(_lib.load().ublr_null_vectors(T.ctypes.data, ell, ptr.ctypes.data, idx.ctypes.data, n,
                                             Z.ctypes.data, res.ctypes.data), "ublr_null_vectors")
    # ||T[rows]||_F per set (the reference's residual scale)
    rn2 = np.einsum("ij,ij->i", T, T)
    seg = np.add.reduceat(rn2[idx], ptr[:-1]) if idx.size else np.zeros(n)
    seg[np.diff(ptr) == 0] = 0.0
    scale = np.maximum(1.0, np.sqrt(seg))
    ok = res <= rtol * scale
    return Z, res, ok


def batched_null_vectors_numpy(T: np.ndarray, rows_list: list, rtol: float = 1e-12):
    """numpy form of batched_null_vectors (the reference's own QR); kept as
    the cross-check for the C-ABI version."""
    ell = T.shape[1]
    n = len(rows_list)
    Z = np.zeros((n, ell))
    res = np.zeros(n)
    ok = np.ones(n, dtype=bool)
    sizes = np.array([len(r) for r in rows_list])
    for sz in np.unique(sizes):
        idx = np.flatnonzero(sizes == sz)
        rows = np.array([rows_list[i] for i in idx], dtype=np.int64)  # (G, sz)
        sub = T[rows]                                                 # (G, sz, ell)
        q = np.linalg.qr(np.transpose(sub, (0, 2, 1)), mode="complete")[0]
        z = q[:, :, ell - 1]
        Z[idx] = z
        r = np.linalg.norm(np.einsum("gij,gj->gi", sub, z), axis=1)
        res[idx] = r
        scale = np.maximum(1.0, np.linalg.norm(sub, axis=(1, 2)))
        ok[idx] = r <= rtol * scale
    return Z, res, ok


def tag_null_vector(T: TaggingMatrix, tess: Tessellation, i: int) -> NullVector:
    """ref/tagging.py:126-139."""
    Z, res, ok = batched_null_vectors(T.entries, [tess.neighbor_lists[i]])
    if not ok[0]:
        raise DegenerateTagsError(f"block {i}: requested null space does not exist")
    limit = 1e-12 * max(1.0, _fro(T.entries))
    if res[0] > limit:
        raise DegenerateTagsError(f"block {i}: null-vector residual {res[0]:.3e} exceeds {limit:.3e}")
    return NullVector(block=i, vector=Z[0], residual=float(res[0]))


def projected_tags(T: TaggingMatrix, tess: Tessellation, nv: NullVector) -> ProjectedTags:
    return ProjectedTags(block=nv.block, values=T.entries @ nv.vector)


def aspect_ratio(pt: ProjectedTags, tess: Tessellation, i: int | None = None) -> float:
    """ref/tagging.py:110-123."""
    block = pt.block if i is None else i
    far = tess.far_fields[block]
    if len(far) == 0:
        raise ValueError(f"block {block} has an empty far field (b too small)")
    mags = np.abs(pt.values[far])
    hi, lo = mags.max(), mags.min()
    if hi == 0.0:
        return 1.0
    if lo == 0.0:
        return float("inf")
    return float(hi / lo)


def null_basis_host(sub: np.ndarray, k: int, rtol: float = 1e-12) -> np.ndarray:
    """ref/linalg.py:72-94 for the tiny host tagging problems: the last k
    columns of numpy's complete QR of sub^T (the reference's own
    orthonormalisation, so nullity >= 2 picks the same directions)."""
    n = sub.shape[1]
    if k > n:
        raise DegenerateTagsError(f"k={k} exceeds column count {n}")
    q = np.linalg.qr(sub.T, mode="complete")[0]
    X = q[:, n - k:]
    if np.linalg.norm(sub @ X) > rtol * max(1.0, np.linalg.norm(sub)):
        raise DegenerateTagsError(f"requested null space of dimension {k} does not exist")
    return X


def _ratio_cols(far_vals: np.ndarray) -> np.ndarray:
    """ref/tagging.py:157-166: aspect ratio of each column of (|F|, n)."""
    mags = np.abs(far_vals)
    hi, lo = mags.max(axis=0), mags.min(axis=0)
    out = np.full(far_vals.shape[1], np.inf)
    np.divide(hi, lo, out=out, where=lo > 0)
    out[hi == 0] = 1.0
    return out


def _golden_min(f, a, b, tol=1e-10, max_iter=200):
    """ref/tagging.py:169-191: golden-section minimisation on [a, b]."""
    g = (np.sqrt(5.0) - 1.0) / 2.0
    x1, x2 = b - g * (b - a), a + g * (b - a)
    f1, f2 = f(x1), f(x2)
    for _ in range(max_iter):
        if b - a < tol:
            break
        if f1 <= f2:
            b, x2, f2 = x2, x1, f1
            x1 = b - g * (b - a)
            f1 = f(x1)
        else:
            a, x1, f1 = x1, x2, f2
            x2 = a + g * (b - a)
            f2 = f(x2)
    return (x1, f1) if f1 <= f2 else (x2, f2)


def _search_circle(P, grid_points):
    """ref/tagging.py:241-262: nullity 2 -- grid over the half circle, then
    golden-section refinement inside the best grid cell."""
    th = np.linspace(0.0, np.pi, grid_points, endpoint=False)
    ratios = _ratio_cols(P @ np.vstack((np.cos(th), np.sin(th))))
    best = int(np.argmin(ratios))
    h = np.pi / grid_points
    t_ref, r_ref = _golden_min(lambda t: _ratio_cols((P @ np.array([np.cos(t), np.sin(t)]))[:, None])[0],
                               th[best] - h, th[best] + h)
    t, r = (t_ref, r_ref) if r_ref <= ratios[best] else (th[best], ratios[best])
    return np.array([np.cos(t), np.sin(t)]), float(r)


def _search_sphere(P, coarse=64, zoom_rounds=3):
    """ref/tagging.py:265-289: nullity >= 3 -- (phi, psi) grid over the
    sphere of the first three null directions with three zoom rounds."""
    phi_c, phi_h, psi_c, psi_h = np.pi / 2, np.pi / 2, np.pi, np.pi
    best_a, best_r = None, np.inf
    n = coarse
    for _ in range(zoom_rounds + 1):
        pp, ss = np.meshgrid(np.linspace(phi_c - phi_h, phi_c + phi_h, n),
                             np.linspace(psi_c - psi_h, psi_c + psi_h, n), indexing="ij")
        pp, ss = pp.ravel(), ss.ravel()
        A = np.column_stack((np.cos(pp), np.sin(pp) * np.cos(ss), np.sin(pp) * np.sin(ss)))
        ratios = _ratio_cols(P @ A.T)
        idx = int(np.argmin(ratios))
        if ratios[idx] < best_r:
            best_r, best_a = float(ratios[idx]), A[idx]
        phi_c, psi_c = pp[idx], ss[idx]
        phi_h /= n / 4.0
        psi_h /= n / 4.0
        n = 17
    return best_a, best_r


def optimize_null_vector(T: TaggingMatrix, tess: Tessellation, i: int, grid_points: int = 4096,
                         base: NullVector | None = None) -> NullVector:
    """ref/tagging.py:194-238: the unit vector of null(T(N_i, :)) with the
    smallest far-field aspect ratio (searched over the first <= 3 null
    directions); the unoptimised vector is kept when it is at least as good.
    Nullity 1 returns the base vector with a warning."""
    if base is None:
        base = tag_null_vector(T, tess, i)
    far, nbrs = tess.far_fields[i], tess.neighbor_lists[i]
    nullity = T.n_cols - len(nbrs)
    if nullity < 2:
        warnings.warn(f"block {i}: null space is one-dimensional, nothing to optimize")
        return base
    if len(far) == 0:
        return base
    sub = T.entries[nbrs, :]
    X = null_basis_host(sub, nullity)[:, :min(nullity, 3)]
    P = T.entries[far, :] @ X
    coeffs, ratio = _search_circle(P, grid_points) if X.shape[1] == 2 else _search_sphere(P)
    if aspect_ratio(projected_tags(T, tess, base), tess) <= ratio:
        return base
    z = X @ coeffs
    z /= np.linalg.norm(z)
    return NullVector(block=i, vector=z, residual=float(np.linalg.norm(sub @ z)))


def _optimize_plan(plan: TaggingPlan, tess: Tessellation) -> TaggingPlan:
    """The optimize=True branch of ref/tagging.py:355-379 over an evaluated
    plan: blocks of nullity >= 2 get optimize_null_vector, every block with a
    far field gets rho_optimized. Host planning only -- the chosen vectors
    feed the same GPU block-QR launch as the base ones."""
    T = plan.matrix
    Z, res = plan.Z.copy(), np.array([nv.residual for nv in plan.null_vectors])
    rho_opt = np.full(tess.b, np.nan)
    nl = np.array([len(x) for x in tess.neighbor_lists])
    for i in range(tess.b):
        far = tess.far_fields[i]
        if T.n_cols - nl[i] >= 2:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                nv = optimize_null_vector(T, tess, i, base=NullVector(i, Z[i], float(res[i])))
            Z[i], res[i] = nv.vector, nv.residual
        if len(far) > 0:
            rho_opt[i] = _ratio_cols((T.entries[far, :] @ Z[i])[:, None])[0]
    return TaggingPlan(matrix=T, null_vectors=NullVectors(Z, res), rho_base=plan.rho_base, rho_optimized=rho_opt,
                       attempts=plan.attempts)


def extra_sample_vectors(plan: TaggingPlan, tess: Tessellation) -> np.ndarray:
    """Per-block combination vectors of tagging_bases(extra_samples=True)
    (ref/bases.py:177-188). The reference concatenates the samples of every
    orthonormal null direction, but U_i = the first k columns of an unpivoted
    QR depends only on the first sample (k <= group width), so
    the GPU path combines with the first column of null_basis(T(N_i,:),
    nullity) where nullity >= 2 and with the plan's z^(i) elsewhere."""
    T = plan.matrix.entries
    Z = plan.Z.copy()
    for i, nb in enumerate(tess.neighbor_lists):
        nullity = T.shape[1] - len(nb)
        if nullity >= 2:
            Z[i] = null_basis_host(T[nb, :], nullity)[:, 0]
    return Z


DEVICE_PLAN_MIN_B = 1024


def _aspect_device(E, Z, tess):
    """rho per block by the C-ABI kernel ublr_tag_aspect (b x b dot products on
    the GPU; the host form below is the CPU-test path)."""
    import torch

    from . import _lib
    from .tessellation import device_tess
    dt = device_tess(tess, torch.device("cuda"))
    Ed, Zd = _lib.h2d(E, dt.device), _lib.h2d(Z, dt.device)
    rho = torch.empty(tess.b, dtype=torch.float64, device=dt.device)
    _lib.call("ublr_tag_aspect", _lib.ptr(Ed), _lib.ptr(Zd), E.shape[1], _lib.ptr(dt.nptr), _lib.ptr(dt.nidx),
              tess.b, _lib.ptr(rho), _lib.stream_handle())
    return rho.cpu().numpy()


def _evaluate(T: TaggingMatrix, tess: Tessellation, attempts: int, device: bool = False) -> TaggingPlan:
    """ref/tagging.py:355-379 for optimize=False, batched: one C-ABI host call
    (ublr_tag_plan_host) for the null vectors, residuals and, unless `device`
    (GPU aspect ratios for large b), the aspect ratios."""
    from . import _lib
    E = np.ascontiguousarray(T.entries, dtype=np.float64)
    b, ell = E.shape
    ptr, idx = _neighbour_csr(tess)
    if len(ptr) > 1 and int(np.diff(ptr).max()) >= ell:
        raise DegenerateTagsError("requested null space of dimension 1 does not exist")
    Z = np.zeros((b, ell))
    res = np.zeros(b)
    scale = np.zeros(b)
    rho = None if device else np.zeros(b)
    _lib.check(_lib.load().ublr_tag_plan_host(E.ctypes.data, ell, ptr.ctypes.data, idx.ctypes.data, b, Z.ctypes.data,
                                              res.ctypes.data, scale.ctypes.data,
                                              None if rho is None else rho.ctypes.data), "ublr_tag_plan_host")
    ok = res <= 1e-12 * scale
    if not ok.all():
        i = int(np.flatnonzero(~ok)[0])
        raise DegenerateTagsError(f"block {i}: requested null space does not exist")
    limit = 1e-12 * max(1.0, _fro(E))
    if (res > limit).any():
        i = int(np.flatnonzero(res > limit)[0])
        raise DegenerateTagsError(f"block {i}: null-vector residual {res[i]:.3e} exceeds {limit:.3e}")
    if device:
        rho = _aspect_device(E, Z, tess)
    return TaggingPlan(matrix=T, null_vectors=NullVectors(Z, res), rho_base=rho, rho_optimized=None,
                       attempts=attempts)


def _evaluate_numpy(T: TaggingMatrix, tess: Tessellation, attempts: int) -> TaggingPlan:
    """The same evaluation with numpy (batched_null_vectors + |T Z^T|): the
    cross-check of ublr_tag_plan_host in the CPU tests."""
    E = T.entries
    Z, res, ok = batched_null_vectors(E, tess.neighbor_lists, csr=_neighbour_csr(tess))
    if not ok.all():
        i = int(np.flatnonzero(~ok)[0])
        raise DegenerateTagsError(f"block {i}: requested null space does not exist")
    limit = 1e-12 * max(1.0, _fro(E))
    if (res > limit).any():
        i = int(np.flatnonzero(res > limit)[0])
        raise DegenerateTagsError(f"block {i}: null-vector residual {res[i]:.3e} exceeds {limit:.3e}")
    b = tess.b
    nvs = NullVectors(Z, res)
    ptr, idx = _neighbour_csr(tess)
    P = np.abs(E @ Z.T)                     # P[j, i] = |<t_j, z^(i)>|
    nl = np.diff(ptr)
    rows_near = idx
    cols_near = np.repeat(np.arange(b), nl)
    far_any = nl < b
    P[rows_near, cols_near] = np.inf        # exclude the near field from the min ...
    lo = P.min(axis=0)
    P[rows_near, cols_near] = -np.inf       # ... and from the max
    hi = P.max(axis=0)
    rho = np.full(b, np.nan)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(hi == 0.0, 1.0, np.where(lo == 0.0, np.inf, hi / lo))
    rho[far_any] = r[far_any]
    return TaggingPlan(matrix=T, null_vectors=nvs, rho_base=rho, rho_optimized=None, attempts=attempts)


def plan_tagging(tess, extra_cols=0, distribution="gaussian", stream=None, optimize=False,
                 max_redraws=5, ratio_limit=1e6, extra_check=None, first=None, device=False) -> TaggingPlan:
    """Redraw policy of ref/tagging.py:306-352. `first` may carry the policy's
    first draw (make_tagging_matrix(..., stream.child(0))) when the caller has
    already made it. `device`: aspect ratios by the GPU kernel; "auto" uses it
    for b >= DEVICE_PLAN_MIN_B (the b x b host product dominates there, ~70 ms
    per draw at b = 4096); False keeps the host form (CPU tests)."""
    if device == "auto":
        device = tess.b >= DEVICE_PLAN_MIN_B
    stream = stream or RandomStream(0)
    last, plan = None, None
    for attempt in range(max_redraws + 1):
        if attempt == 0 and first is not None:
            T = first
        else:
            T = make_tagging_matrix(tess.b, tess.dim, extra_cols, distribution, stream.child(attempt))
        if extra_check is not None and not extra_check(T):
            last = DegenerateTagsError("extra_check rejected the draw")
            continue
        try:
            plan = _evaluate(T, tess, attempt + 1, device=device)
            if optimize:
                plan = _optimize_plan(plan, tess)
        except DegenerateTagsError as exc:
            last = exc
            continue
        eff = plan.rho_optimized if plan.rho_optimized is not None else plan.rho_base
        fin = eff[~np.isnan(eff)]
        worst = fin.max() if fin.size else 1.0
        if np.isfinite(worst) and worst <= ratio_limit:
            return plan
    if plan is None:
        raise DegenerateTagsError(f"no usable tagging matrix after {max_redraws + 1} draws: {last}")
    warnings.warn(f"tagging matrix still has aspect ratio above {ratio_limit:.0e} after "
                  f"{max_redraws + 1} draws; proceeding with the last one")
    return plan


def pair_vectors(T_entries: np.ndarray, tess: Tessellation, denom_rtol: float = 1e-10):
    """Per near pair p = (i, j) in neighbour-CSR order: unit null vector of
    T(N_i \\ {j}, :) and denominator <t_j, z> (ref/reconstruction.py:344-355).
    Raises DegenerateTagsError like the reference."""
    limit = denom_rtol * max(1.0, _fro(T_entries))
    sets, excl = [], []
    for i, nb in enumerate(tess.neighbor_lists):
        for j in nb:
            sets.append([r for r in nb if r != j])
            excl.append(j)
    Z, res, ok = batched_null_vectors(T_entries, sets)
    if not ok.all():
        raise DegenerateTagsError("requested null space of dimension 1 does not exist")
    den = np.einsum("pj,pj->p", T_entries[np.array(excl)], Z)
    if (np.abs(den) < limit).any():
        raise DegenerateTagsError("projected tag for a near pair vanished")
    return Z, den


def b2_denominators_ok(T, tess: Tessellation, rtol: float = 1e-10) -> bool:
    """ref/reconstruction.py:310-323."""
    entries = T.entries if isinstance(T, TaggingMatrix) else np.asarray(T)
    try:
        pair_vectors(entries, tess, rtol)
    except DegenerateTagsError:
        return False
    return True
