"""Seeded streams and dense helpers (mirror of ref/linalg.py:14-139).

`RandomStream` keeps the reference's semantics exactly (numpy Philox keyed
by SeedSequence(seed, spawn_key=key), row-major `standard_normal`); its host
methods serve host-side planning (the b x ell tagging matrix). Every test
matrix of the compression itself is drawn on the GPU by
`device_normals` (C-ABI `ublr_rng_normals`, bit-identical to numpy).
"""

from __future__ import annotations

import numpy as np

from . import _lib


class RandomStream:
    """ref/linalg.py:14-45."""

    def __init__(self, seed: int, key: tuple = ()):
        self.seed = int(seed)
        self.key = tuple(int(i) for i in key)
        self._gen = None

    def child(self, *indices: int) -> "RandomStream":
        return RandomStream(self.seed, self.key + indices)

    @property
    def generator(self) -> np.random.Generator:
        if self._gen is None:
            seq = np.random.SeedSequence(self.seed, spawn_key=self.key)
            self._gen = np.random.Generator(np.random.Philox(seq))
        return self._gen

    def philox_key(self) -> tuple:
        """128-bit Philox key (numpy derives it as SeedSequence.generate_state(2, uint64))."""
        st = np.random.SeedSequence(self.seed, spawn_key=self.key).generate_state(2, np.uint64)
        return int(st[0]), int(st[1])

    def normal(self, rows: int, cols: int) -> np.ndarray:
        return self.generator.standard_normal((rows, cols))

    def uniform(self, rows: int, cols: int) -> np.ndarray:
        return self.generator.random((rows, cols))

    def __repr__(self):
        return f"RandomStream(seed={self.seed}, key={self.key})"


def gaussian(rows: int, cols: int, stream: RandomStream) -> np.ndarray:
    """ref/linalg.py:48-52 (host array, bit-identical to the reference)."""
    if rows < 0 or cols < 0:
        raise ValueError("matrix dimensions must be nonnegative")
    return stream.normal(rows, cols)


def device_normals(specs, out):
    """Fill `out` (a CUDA float64 tensor) from several Gaussian streams.

    specs: iterable of (stream, rows, cols, out_offset, ld, rowmap) where
    normal n of the stream lands at out.flat[out_offset + row(n) * ld + n % cols]
    with row(n) = rowmap[n // cols] (rowmap: CUDA int32 tensor or None).
    The same numbers numpy's `stream.normal(rows, cols)` returns.
    """
    import torch

    _lib.require_device()
    specs = list(specs)
    if not specs:
        return out
    from .seedseq import philox_keys

    ns = len(specs)
    rec = np.zeros(ns, dtype=_lib.RNG_STREAM_DTYPE)
    by_seed = {}
    for s, sp in enumerate(specs):
        by_seed.setdefault(sp[0].seed, []).append(s)
    for seed, idx in by_seed.items():   # vectorised SeedSequence (bit-identical to numpy's)
        kk = philox_keys(seed, [specs[s][0].key for s in idx])
        rec["key0"][idx] = kk[:, 0]
        rec["key1"][idx] = kk[:, 1]
    rows = np.array([sp[1] for sp in specs], dtype=np.int64)
    cols = np.array([sp[2] for sp in specs], dtype=np.int64)
    counts = rows * cols
    rec["count"] = counts
    rec["cols"] = np.maximum(cols, 1)
    rec["ld"] = [sp[4] for sp in specs]
    rec["out_offset"] = [sp[3] for sp in specs]
    rec["rowmap"] = [_lib.ptr(sp[5]) for sp in specs]
    keep = [sp[5] for sp in specs if sp[5] is not None]
    lib = _lib.load()
    ws_bytes = int(lib.ublr_rng_workspace_bytes(counts.ctypes.data, len(specs)))
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=out.device)
    rec_d = _lib.h2d(rec.view(np.uint8), out.device)
    _lib.call("ublr_rng_normals", _lib.ptr(rec_d), counts.ctypes.data, len(specs), _lib.ptr(out),
              _lib.ptr(ws), ws_bytes, _lib.stream_handle(), launches=_lib.rng_launches(counts))
    # keep host/device descriptors alive until the stream has consumed them
    out._ublr_keepalive = (rec_d, ws, keep)
    return out


def device_normals_keys(seed, keys, rows, cols, offsets, ld, rowmap, out, suffix=None):
    """Vectorised form of device_normals for many streams of one seed:
    stream s is RandomStream(seed, keys[s]) with rows[s] x cols normals at
    out.flat[offsets[s] + r * ld + c] (rowmap shared by all streams or None).
    With `suffix` ((n, ns) ints), `keys` is one prefix tuple and stream s is
    RandomStream(seed, keys + tuple(suffix[s])); the keys are derived by the
    C-ABI host function ublr_seedseq_keys."""

    _lib.require_device()
    launch_normals(rng_launch_record(seed, keys, rows, cols, offsets, ld, rowmap, out.device, suffix), out)
    return out


def rng_launch_record(seed, keys, rows, cols, offsets, ld, rowmap, device, suffix=None):
    """Device stream records + workspace of a device_normals_keys launch set.
    They are a pure function of the arguments: built and uploaded once, the
    normals are drawn on every launch_normals call."""
    from .seedseq import philox_keys, philox_keys_suffixed

    cols_a = np.broadcast_to(np.asarray(cols, dtype=np.int64), np.shape(rows))   # scalar or per stream
    ld_a = np.broadcast_to(np.asarray(ld, dtype=np.int64), np.shape(rows))
    ck = (int(seed), tuple(keys) if suffix is not None else tuple(map(tuple, keys)),
          np.asarray(rows, dtype=np.int64).tobytes(), cols_a.tobytes(), np.asarray(offsets, dtype=np.int64).tobytes(),
          ld_a.tobytes(), _lib.ptr(rowmap), None if suffix is None else np.asarray(suffix).tobytes(), str(device))
    hit = _RNG_CACHE.get(ck)
    if hit is not None:
        return hit
    if suffix is not None:
        kk = philox_keys_suffixed(seed, keys, suffix)
    else:
        kk = philox_keys(seed, keys)
    ns = kk.shape[0]
    rec = np.zeros(ns, dtype=_lib.RNG_STREAM_DTYPE)
    rec["key0"], rec["key1"] = kk[:, 0], kk[:, 1]
    counts = np.asarray(rows, dtype=np.int64) * cols_a
    rec["count"] = counts
    rec["cols"] = np.maximum(cols_a, 1)
    rec["ld"] = ld_a
    rec["out_offset"] = np.asarray(offsets, dtype=np.int64)
    rec["rowmap"] = _lib.ptr(rowmap)
    lib = _lib.load()
    ws_bytes = int(lib.ublr_rng_workspace_bytes(counts.ctypes.data, ns))
    import torch
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device=device)
    rec_d = _lib.h2d(rec.view(np.uint8), device)
    if len(_RNG_CACHE) > 64:
        _RNG_CACHE.clear()
    # the launch arguments as plain ints, resolved once (the RNG launch is the
    # first thing a compression queues: its host latency is on the step's
    # critical path)
    fast = (_lib.ptr(rec_d), counts.ctypes.data, ns, _lib.ptr(ws), ws_bytes, _lib.rng_launches(counts))
    hit = _RNG_CACHE[ck] = (rec_d, counts, ns, ws, ws_bytes, rowmap, fast)
    return hit


def launch_normals(record, out, out_ptr=None):
    """Draw the normals of a rng_launch_record into `out` (K1); `out_ptr`
    overrides the destination pointer."""
    rp, cp, ns, wp, ws_bytes, launches = record[6]
    _lib.call("ublr_rng_normals", rp, cp, ns, _lib.ptr(out) if out_ptr is None else out_ptr, wp, ws_bytes,
              _lib.stream_handle(), launches=launches)
    return out


_RNG_CACHE = {}


def col_basis(B, k: int) -> np.ndarray:
    """ref/linalg.py:55-69 on the GPU (Householder QR kernel K4)."""
    import torch

    B = np.asarray(B, dtype=float)
    m, n = B.shape
    if k > min(m, n):
        raise ValueError(f"k={k} exceeds matrix dimensions {m}x{n}")
    if k == 0:
        return np.zeros((m, 0))
    _lib.require_device()
    dev = torch.device("cuda")
    Bd = torch.from_numpy(np.ascontiguousarray(B)).to(dev)
    off = torch.tensor([0, m], dtype=torch.int32, device=dev)
    col0 = torch.zeros(1, dtype=torch.int32, device=dev)
    Q = torch.empty((m, k), dtype=torch.float64, device=dev)
    # mode 1 (sample = columns col0..) | 2 (plain QR: no identity shortcut for k == m)
    _lib.call("ublr_block_qr", _lib.ptr(Bd), n, 3, None, 0, 0, _lib.ptr(col0), _lib.ptr(off), 1, k,
              _lib.ptr(Q), k, _lib.stream_handle(), m)
    return Q.cpu().numpy()
