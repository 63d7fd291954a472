"""UBLR1 binary container for compressed representations (ref/container.py:1-114).

Same byte layout as the reference (little-endian u64 integers, f64 values,
row-major dense blocks), so files are interchangeable both ways:

    magic "UBLR1"
    n, b, k, d, tess_json_len, n_b_blocks
    tess_json   (json.dumps(sort_keys, compact) of dim, b, blocks, neighbors,
                 colors; ids 1-based)
    effective ranks, one per block
    U blocks in block order, then V blocks
    core (K x K)
    B index table: (i, j) pairs, 1-based, sorted
    B blocks in table order

`write_ublr` streams a device-resident UniformBLR to disk: U and V are
written straight from their device layout (block i's rows are contiguous in
the permuted order, so with equal ranks the U section is one copy), the core
and the near blocks go through a double-buffered pinned staging area in
fixed-size panels (c5's core is 309 GB; it never has to fit in host memory),
and the D2H copy of panel t+1 overlaps the file write of panel t. Writing the
same representation twice gives identical bytes (ref tests/test_container.py:
32-37). `write_ublr_host` writes host arrays (the CPU path the reference's
files are checked against). `read_ublr` returns a device UniformBLR.
"""

from __future__ import annotations

import json

import numpy as np

from .tessellation import Tessellation, color_boxes

MAGIC = b"UBLR1"
PANEL_BYTES = 256 << 20


def _u64(*values) -> bytes:
    return np.asarray(values, dtype="<u8").tobytes()


def _tess_json(tess: Tessellation) -> bytes:
    return json.dumps(tess.to_json_dict(colors=color_boxes(tess).colors), sort_keys=True,
                      separators=(",", ":")).encode()


def _header(fh, n, tess, rank, n_pairs, ranks):
    tj = _tess_json(tess)
    fh.write(MAGIC)
    fh.write(_u64(n, tess.b, rank, tess.dim, len(tj), n_pairs))
    fh.write(tj)
    fh.write(_u64(*[int(r) for r in ranks]))


def write_ublr_host(path, tess: Tessellation, rank: int, ranks, u_blocks, v_blocks, core, b_blocks: dict) -> None:
    """Host-array writer (ref/container.py:38-58 layout)."""
    pairs = sorted(b_blocks)
    with open(path, "wb") as fh:
        _header(fh, tess.n_points, tess, rank, len(pairs), ranks)
        for blk in list(u_blocks) + list(v_blocks):
            fh.write(np.ascontiguousarray(blk, dtype="<f8").tobytes())
        fh.write(np.ascontiguousarray(core, dtype="<f8").tobytes())
        for i, j in pairs:
            fh.write(_u64(i + 1, j + 1))
        for pq in pairs:
            fh.write(np.ascontiguousarray(b_blocks[pq], dtype="<f8").tobytes())


class _Stager:
    """Double-buffered pinned staging of device tensors into a file."""

    def __init__(self, fh, panel_bytes=PANEL_BYTES):
        import torch
        self.torch = torch
        self.fh = fh
        self.n = max(1, panel_bytes // 8)
        self.buf = [torch.empty(self.n, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        self.ev = [torch.cuda.Event(), torch.cuda.Event()]
        self.pending = [None, None]
        self.slot = 0
        self.stream = torch.cuda.Stream()

    def _flush(self, s):
        if self.pending[s] is not None:
            self.ev[s].synchronize()
            self.fh.write(self.buf[s][:self.pending[s]].numpy().tobytes())
            self.pending[s] = None

    def put(self, flat):
        """Queue a contiguous 1-D float64 device tensor."""
        torch = self.torch
        self.stream.wait_stream(torch.cuda.current_stream())
        for a in range(0, flat.numel(), self.n):
            s = self.slot
            self._flush(s)
            part = flat[a:a + self.n]
            # the source may be a temporary of the caller's stream (a per-block
            # .contiguous()): keep its memory out of the allocator's reuse
            # until this stream's copy has read it
            part.record_stream(self.stream)
            with torch.cuda.stream(self.stream):
                self.buf[s][:part.numel()].copy_(part, non_blocking=True)
                self.ev[s].record(self.stream)
            self.pending[s] = part.numel()
            self.slot ^= 1

    def close(self):
        for _ in range(2):
            self._flush(self.slot)
            self.slot ^= 1


def write_ublr(path, rep) -> None:
    """Stream a device UniformBLR (reconstruction.UniformBLR) to `path`."""
    dt = rep.dt
    ranks = rep.effective_ranks
    with open(path, "wb") as fh:
        _header(fh, rep.n, rep.tess, rep.rank, dt.n_pairs, ranks)
        st = _Stager(fh)
        for M in (rep.U, rep.V):
            if M.shape[1] == 0:
                continue
            if (ranks == M.shape[1]).all() and M.is_contiguous():
                st.put(M.reshape(-1))
            else:
                for i in range(dt.b):
                    st.put(M[dt.off_h[i]:dt.off_h[i + 1], :ranks[i]].contiguous().reshape(-1))
        st.put(rep.core_d.reshape(-1))
        st.close()
        pairs = np.stack([dt.pair_i_h.astype(np.uint64) + 1, dt.nidx_h.astype(np.uint64) + 1], axis=1)
        fh.write(pairs.astype("<u8").tobytes())
        st.put(rep.B_d.reshape(-1))
        st.close()


def read_ublr(path):
    """Container -> device UniformBLR (ref/container.py:61-98)."""
    import torch

    from .reconstruction import UniformBLR
    from .tessellation import device_tess

    with open(path, "rb") as fh:
        raw = fh.read()
    if raw[:len(MAGIC)] != MAGIC:
        raise ValueError(f"{path}: not a UBLR container")
    off = len(MAGIC)

    def take_u64(count):
        nonlocal off
        vals = np.frombuffer(raw, dtype="<u8", count=count, offset=off)
        off += 8 * count
        return vals.astype(np.int64)

    def take_f64(count):
        nonlocal off
        vals = np.frombuffer(raw, dtype="<f8", count=count, offset=off)
        off += 8 * count
        return vals

    n, b, k, d, json_len, n_pairs = (int(x) for x in take_u64(6))
    tj = json.loads(raw[off:off + json_len].decode())
    off += json_len
    blocks = [np.asarray(x, dtype=np.int64) - 1 for x in tj["blocks"]]
    nbrs = [[int(j) - 1 for j in x] for x in tj["neighbors"]]
    tess = Tessellation(dim=int(tj["dim"]), axis_count=0, n_points=n, blocks=blocks, neighbor_lists=nbrs,
                        grid_coords=np.zeros((len(blocks), int(tj["dim"])), dtype=np.int64), full_grid=False)
    if "colors" in tj:
        tess.colors = np.asarray(tj["colors"], dtype=np.int64) - 1
    ranks = take_u64(b)
    dev = torch.device("cuda")
    dt = device_tess(tess, dev)
    if not np.array_equal(ranks, dt.ranks(k)):
        raise ValueError(f"{path}: effective ranks are not min(k, m_i)")
    sizes = dt.sizes
    kk = max(k, 1)
    UV = []
    for _ in range(2):
        M = np.zeros((n, kk))
        for i in range(b):
            M[dt.off_h[i]:dt.off_h[i + 1], :ranks[i]] = take_f64(sizes[i] * ranks[i]).reshape(sizes[i], ranks[i])
        UV.append(torch.from_numpy(M).to(dev))
    K = int(ranks.sum())
    core = torch.from_numpy(take_f64(K * K).reshape(K, K).copy()).to(dev)
    pairs = take_u64(2 * n_pairs).reshape(n_pairs, 2) - 1
    if not (np.array_equal(pairs[:, 0], dt.pair_i_h) and np.array_equal(pairs[:, 1], dt.nidx_h)):
        raise ValueError(f"{path}: near-block table does not match the tessellation's neighbour pairs")
    B = torch.from_numpy(take_f64(int(dt.b_off_h[-1])).copy()).to(dev)
    return UniformBLR(tess, int(k), UV[0], UV[1], core, B, dt, {"source": str(path)})
