"""Vectorised numpy SeedSequence -> Philox key derivation.

numpy keys `Philox(SeedSequence(seed, spawn_key=key))` with
`SeedSequence.generate_state(2, uint64)` (the reference's RandomStream,
ref/linalg.py:30-35). The reference derives one key per test block (2b
streams per compression); doing that through SeedSequence objects costs
~12 us each on the host, i.e. ~0.1 s at b = 4096. This module restates
numpy's published SeedSequence algorithm (O'Neill's seed_seq hash mixing,
numpy/random/bit_generator.pyx: pool of 4 uint32 words, hashmix / mix with
the INIT_A/MULT_A, INIT_B/MULT_B and MIX_MULT_L/R constants) over many spawn
keys at once with uint32 numpy arithmetic. Checked bit-for-bit against
numpy in tests/test_host.py.
"""

from __future__ import annotations

import numpy as np

_INIT_A = np.uint32(0x43B0D7E5)
_MULT_A = np.uint32(0x931E8875)
_INIT_B = np.uint32(0x8B51F9DD)
_MULT_B = np.uint32(0x58F38DED)
_MIX_L = np.uint32(0xCA01F9DD)
_MIX_R = np.uint32(0x4973F715)
_XSHIFT = np.uint32(16)
_POOL = 4


def _words(v: int) -> list:
    """numpy's _coerce_to_uint32_array for a non-negative int."""
    if v < 0:
        raise ValueError("expected non-negative integer")
    if v == 0:
        return [0]
    out = []
    while v > 0:
        out.append(v & 0xFFFFFFFF)
        v >>= 32
    return out


def philox_keys(seed: int, keys) -> np.ndarray:
    """(n, 2) uint64 Philox keys of RandomStream(seed, key) for each key."""
    keys = [tuple(int(x) for x in k) for k in keys]
    n = len(keys)
    out = np.zeros((n, 2), dtype=np.uint64)
    if n == 0:
        return out
    run = _words(int(seed))
    # group keys with identical entropy layout (same word counts): {nspawn: (indices, spawn words)}
    groups = {}
    lens = {len(k) for k in keys}
    if len(lens) == 1:
        arr = np.array(keys, dtype=np.int64).reshape(n, -1)
        if arr.size == 0 or (arr.min() >= 0 and arr.max() < 2 ** 32):
            # every component is a single uint32 word: vectorised fast path
            groups[arr.shape[1]] = (np.arange(n), arr.astype(np.uint32))
    if not groups:
        tmp = {}
        for idx, k in enumerate(keys):
            spawn = [w for x in k for w in _words(x)]
            tmp.setdefault(len(spawn), []).append((idx, spawn))
        groups = {ln: (np.array([i for i, _ in it]), np.array([sp for _, sp in it], dtype=np.uint32).reshape(len(it), ln))
                  for ln, it in tmp.items()}
    with np.errstate(over="ignore"):
        for nspawn, (idxs, spawn) in groups.items():
            r = list(run)
            if nspawn > 0 and len(r) < _POOL:
                r = r + [0] * (_POOL - len(r))
            ent = np.hstack([np.tile(np.array(r, dtype=np.uint32), (len(idxs), 1)), spawn])  # (G, L)
            G, L = ent.shape
            hc = np.full(G, _INIT_A, dtype=np.uint32)

            def hashmix(v):
                nonlocal hc
                v = v ^ hc
                hc = hc * _MULT_A
                v = v * hc
                return v ^ (v >> _XSHIFT)

            def mix(x, y):
                res = _MIX_L * x - _MIX_R * y
                return res ^ (res >> _XSHIFT)

            pool = np.zeros((G, _POOL), dtype=np.uint32)
            for i in range(_POOL):
                v = ent[:, i] if i < L else np.zeros(G, dtype=np.uint32)
                pool[:, i] = hashmix(v)
            for s in range(_POOL):
                for d in range(_POOL):
                    if s != d:
                        pool[:, d] = mix(pool[:, d], hashmix(pool[:, s]))
            for s in range(_POOL, L):
                for d in range(_POOL):
                    pool[:, d] = mix(pool[:, d], hashmix(ent[:, s]))
            # generate_state(2, uint64): 4 uint32 words cycling over the pool
            hb = np.full(G, _INIT_B, dtype=np.uint32)
            st = np.zeros((G, 4), dtype=np.uint32)
            for i in range(4):
                v = pool[:, i % _POOL] ^ hb
                hb = hb * _MULT_B
                v = v * hb
                st[:, i] = v ^ (v >> _XSHIFT)
            k64 = st.astype(np.uint64)
            res = k64[:, 0::2] | (k64[:, 1::2] << np.uint64(32))
            out[idxs] = res
    return out


def _word_list(values) -> list:
    out = []
    for v in values:
        out.extend(_words(int(v)))
    return out


def philox_keys_suffixed(seed: int, prefix, suffix) -> np.ndarray:
    """(n, 2) uint64 Philox keys of RandomStream(seed, prefix + tuple(suffix[s]))
    through the C-ABI host function (the per-compression key derivation of the
    product path; philox_keys above is the numpy restatement it is checked
    against). suffix: (n, ns) array of components < 2**32."""
    from . import _lib

    suffix = np.ascontiguousarray(suffix, dtype=np.int64)
    if suffix.ndim != 2:
        raise ValueError("suffix must be (n, ns)")
    if suffix.size and (suffix.min() < 0 or suffix.max() >= 2 ** 32):
        raise ValueError("suffix components must be uint32 words")
    run = np.array(_words(int(seed)), dtype=np.uint32)
    pre = np.array(_word_list(prefix), dtype=np.uint32)
    suf = suffix.astype(np.uint32)
    n = suf.shape[0]
    out = np.zeros((n, 2), dtype=np.uint64)
    _lib.check(_lib.load().ublr_seedseq_keys(run.ctypes.data, len(run), pre.ctypes.data if len(pre) else None,
                                             len(pre), suf.ctypes.data if suf.size else None, suf.shape[1], n,
                                             out.ctypes.data), "ublr_seedseq_keys")
    return out
