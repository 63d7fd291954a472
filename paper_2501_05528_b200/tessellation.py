"""Flat box partitions (host) and their device layout.

Same public surface and semantics as ref/tessellation.py:20-238
(PointCloud, grid_points, random_points, Tessellation, build_tessellation,
color_boxes, suggest_block_count). Neighbour lists are found by hashing
grid cells (O(b 3^d)) instead of the reference's O(b^2) scan.

`DeviceTess` is the B200 layout of a tessellation: points renumbered
block-contiguously (block i owns permuted rows off[i]:off[i+1], within-block
order = the reference's ascending global order), neighbour CSR (which is the
reference's sorted (i, j) pair order), colour CSR, rank offsets.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_VALID_DIMS = (1, 2, 3)


@dataclass(frozen=True)
class PointCloud:
    """Points in [0,1]^d (ref/tessellation.py:20-41)."""

    coords: np.ndarray
    dim: int

    def __post_init__(self):
        c = np.atleast_2d(np.asarray(self.coords, dtype=float))
        object.__setattr__(self, "coords", c)
        if self.dim not in _VALID_DIMS:
            raise ValueError(f"invalid dimension d={self.dim}, expected 1, 2, or 3")
        if c.ndim != 2 or c.shape[1] != self.dim:
            raise ValueError(f"coords must have shape (n, {self.dim})")
        if c.shape[0] < 1:
            raise ValueError("point cloud must contain at least one point")
        if np.any(c < 0.0) or np.any(c > 1.0):
            raise ValueError("points must lie inside the unit hypercube [0,1]^d")

    @property
    def n(self) -> int:
        return self.coords.shape[0]


def grid_points(per_axis: int, d: int) -> PointCloud:
    """Cell-centre grid, meshgrid 'ij' order (ref/tessellation.py:44-49)."""
    centres = (np.arange(per_axis) + 0.5) / per_axis
    mesh = np.meshgrid(*([centres] * d), indexing="ij")
    return PointCloud(np.stack([a.ravel() for a in mesh], axis=1), d)


def random_points(n: int, d: int, stream) -> PointCloud:
    """Uniform points from a RandomStream (ref/tessellation.py:52-54)."""
    return PointCloud(stream.uniform(n, d), d)


@dataclass
class BoxColoring:
    colors: np.ndarray
    num_colors: int


@dataclass
class Tessellation:
    """ref/tessellation.py:57-116."""

    dim: int
    axis_count: int
    n_points: int
    blocks: list
    neighbor_lists: list
    grid_coords: np.ndarray
    full_grid: bool
    points: PointCloud | None = None
    colors: np.ndarray | None = None   # stored colouring (read from a UBLR1 container), else computed
    _far_fields: list = field(default=None, repr=False)
    _device: dict = field(default_factory=dict, repr=False)

    @property
    def b(self) -> int:
        return len(self.blocks)

    @property
    def block_sizes(self) -> np.ndarray:
        return np.array([len(x) for x in self.blocks])

    @property
    def max_block_size(self) -> int:
        return int(self.block_sizes.max())

    @property
    def far_fields(self) -> list:
        if self._far_fields is None:
            allb = np.arange(self.b)
            self._far_fields = [np.setdiff1d(allb, nb).tolist() for nb in self.neighbor_lists]
        return self._far_fields

    def neighbor_row_count(self, i: int) -> int:
        return int(sum(len(self.blocks[j]) for j in self.neighbor_lists[i]))

    def neighbor_indices(self, i: int) -> np.ndarray:
        return np.concatenate([self.blocks[j] for j in self.neighbor_lists[i]])

    def to_json_dict(self, colors=None) -> dict:
        out = {"dim": self.dim, "b": self.b,
               "blocks": [(np.asarray(x) + 1).tolist() for x in self.blocks],
               "neighbors": [[j + 1 for j in nb] for nb in self.neighbor_lists]}
        if colors is not None:
            out["colors"] = [int(c) + 1 for c in np.asarray(colors)]
        return out


def suggest_block_count(n: int, k: int, d: int) -> int:
    """ref/tessellation.py:127-140."""
    if n < 1 or k < 1:
        raise ValueError("n and k must be positive")
    if d not in _VALID_DIMS:
        raise ValueError(f"invalid dimension d={d}")
    per_axis = int(np.floor((np.sqrt(3.0 ** d / k) * np.sqrt(n)) ** (1.0 / d) + 0.5))
    return max(per_axis, 2) ** d


def _per_axis(target: int, d: int) -> int:
    if target < 1:
        raise ValueError("target_block_count must be positive")
    guess = int(round(target ** (1.0 / d)))
    for c in (guess - 1, guess, guess + 1):
        if c >= 1 and c ** d == target:
            return c
    raise ValueError(f"target_block_count={target} is not a {d}-th power of a per-axis count")


def build_tessellation(points: PointCloud, target_block_count: int) -> Tessellation:
    """Regular grid of boxes, empty cells dropped (ref/tessellation.py:143-185)."""
    d = points.dim
    per = _per_axis(target_block_count, d)
    cell = np.minimum((points.coords * per).astype(np.int64), per - 1)
    flat = np.zeros(points.n, dtype=np.int64)
    for a in range(d):
        flat = flat * per + cell[:, a]
    order = np.argsort(flat, kind="stable")       # stable: ascending indices per cell
    sflat = flat[order]
    starts = np.flatnonzero(np.r_[True, sflat[1:] != sflat[:-1]])
    occupied = sflat[starts]
    blocks = [np.asarray(g) for g in np.split(order, starts[1:])]
    b = len(blocks)
    grid = np.zeros((b, d), dtype=np.int64)
    rem = occupied.copy()
    for a in range(d - 1, -1, -1):
        grid[:, a] = rem % per
        rem //= per
    # neighbour lists by cell hashing: box id of every occupied cell
    box_of_cell = {int(c): i for i, c in enumerate(occupied)}
    offsets = np.stack(np.meshgrid(*([np.arange(-1, 2)] * d), indexing="ij"), -1).reshape(-1, d)
    nbrs = []
    for i in range(b):
        cand = grid[i] + offsets
        ok = np.all((cand >= 0) & (cand < per), axis=1)
        ids = []
        for c in cand[ok]:
            f = 0
            for a in range(d):
                f = f * per + int(c[a])
            j = box_of_cell.get(f)
            if j is not None:
                ids.append(j)
        nbrs.append(sorted(ids))
    return Tessellation(dim=d, axis_count=per, n_points=points.n, blocks=blocks, neighbor_lists=nbrs,
                        grid_coords=grid, full_grid=(b == per ** d), points=points)


def color_boxes(tess: Tessellation) -> BoxColoring:
    """Distance-2 colouring (ref/tessellation.py:188-219); cached on the
    tessellation (a pure function of it)."""
    cached = tess._device.get("color_boxes")
    if cached is not None:
        return cached
    out = _color_boxes(tess)
    tess._device["color_boxes"] = out
    return out


def _color_boxes(tess: Tessellation) -> BoxColoring:
    if tess.colors is not None:
        colours = np.asarray(tess.colors, dtype=np.int64)
        return BoxColoring(colors=colours, num_colors=int(colours.max()) + 1)
    if tess.full_grid:
        code = np.zeros(tess.b, dtype=np.int64)
        for a in range(tess.dim):
            code = code * 3 + tess.grid_coords[:, a] % 3
        colours = np.unique(code, return_inverse=True)[1].ravel()
    else:
        sets = [set(nb) for nb in tess.neighbor_lists]
        colours = np.full(tess.b, -1, dtype=np.int64)
        for i in range(tess.b):
            taken = {colours[j] for j in range(tess.b)
                     if j != i and colours[j] >= 0 and sets[i] & sets[j]}
            c = 0
            while c in taken:
                c += 1
            colours[i] = c
    return BoxColoring(colors=colours, num_colors=int(colours.max()) + 1)


class DeviceTess:
    """Device-resident layout of a tessellation (see module docstring)."""

    def __init__(self, tess: Tessellation, device):
        import torch

        self.tess = tess
        self.device = device
        b = tess.b
        sizes = tess.block_sizes.astype(np.int64)
        self.b = b
        self.n = tess.n_points
        self.sizes = sizes
        self.m_max = int(sizes.max())
        self.off_h = np.concatenate(([0], np.cumsum(sizes))).astype(np.int32)
        self.perm_h = np.concatenate(tess.blocks).astype(np.int32)
        self.inv_h = np.empty_like(self.perm_h)
        self.inv_h[self.perm_h] = np.arange(self.n, dtype=np.int32)
        nlen = np.array([len(x) for x in tess.neighbor_lists], dtype=np.int64)
        self.nptr_h = np.concatenate(([0], np.cumsum(nlen))).astype(np.int32)
        self.nidx_h = np.concatenate([np.asarray(x, dtype=np.int32) for x in tess.neighbor_lists])
        self.pair_i_h = np.repeat(np.arange(b, dtype=np.int32), nlen)
        self.n_pairs = int(len(self.nidx_h))
        pos = {(int(i), int(j)): q for q, (i, j) in enumerate(zip(self.pair_i_h, self.nidx_h))}
        # tpair[q]: index of the transposed pair (nidx[q], pair_i[q])
        self.tpair_h = np.array([pos[(int(j), int(i))] for i, j in zip(self.pair_i_h, self.nidx_h)], dtype=np.int32)
        bsz = sizes[self.pair_i_h] * sizes[self.nidx_h]
        self.b_off_h = np.concatenate(([0], np.cumsum(bsz))).astype(np.int64)
        col = color_boxes(tess)
        self.colours_h = np.asarray(col.colors, dtype=np.int32)
        self.n_colours = col.num_colors
        order = np.argsort(self.colours_h, kind="stable")
        counts = np.bincount(self.colours_h, minlength=self.n_colours)
        self.cptr_h = np.concatenate(([0], np.cumsum(counts))).astype(np.int32)
        self.cidx_h = order.astype(np.int32)
        # pair_of[i, c]: the near pair (i, j) with colour(j) = c, or -1; None if
        # a neighbourhood repeats a colour (invalid colouring, see _check_coloring)
        key = self.pair_i_h.astype(np.int64) * self.n_colours + self.colours_h[self.nidx_h]
        if np.unique(key).size == key.size:
            po = np.full(b * self.n_colours, -1, dtype=np.int32)
            po[key] = np.arange(self.n_pairs, dtype=np.int32)
            self.pair_of_h = po
        else:
            self.pair_of_h = None

        def t(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(device)

        self.off = t(self.off_h)
        self.perm = t(self.perm_h)
        self.inv = t(self.inv_h)
        self.nptr = t(self.nptr_h)
        self.nidx = t(self.nidx_h)
        self.pair_i = t(self.pair_i_h)
        self.tpair = t(self.tpair_h)
        self.b_off = t(self.b_off_h)
        self.colours = t(self.colours_h)
        self.cptr = t(self.cptr_h)
        self.cidx = t(self.cidx_h)
        self.pair_of = None if self.pair_of_h is None else t(self.pair_of_h)
        self._roff = {}
        self.rng_records = {}   # memoised launch records of the test-block draws (bases.draw_test_pair)

    def ranks(self, k: int) -> np.ndarray:
        return np.minimum(k, self.sizes)

    def roff(self, k: int):
        """(host, device) rank offsets for rank k (ref/bases.py:63-65)."""
        if k not in self._roff:
            import torch
            h = np.concatenate(([0], np.cumsum(self.ranks(k)))).astype(np.int32)
            self._roff[k] = (h, torch.from_numpy(h).to(self.device))
        return self._roff[k]

    def to_perm_rows(self, X):
        """Host (N x w, original order) -> device (N x w, permuted rows)."""
        import torch
        Xt = torch.as_tensor(np.ascontiguousarray(X, dtype=np.float64))
        return Xt.to(self.device)[self.perm.long()].contiguous()

    def from_perm_rows(self, Xd):
        """Device (permuted rows) -> host numpy in original order."""
        out = np.empty(tuple(Xd.shape), dtype=np.float64)
        out[self.perm_h] = Xd.cpu().numpy()
        return out


def device_tess(tess: Tessellation, device) -> DeviceTess:
    key = str(device)
    if key not in tess._device:
        tess._device[key] = DeviceTess(tess, device)
    return tess._device[key]
