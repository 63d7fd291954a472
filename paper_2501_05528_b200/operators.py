"""Operator plug-in boundary (mirror of ref/operators.py:24-149).

The reference's compressor only touches A through `shape`, `apply(X)` and
`apply_adjoint(X)` on column blocks; any object with those works here too.
The GPU operators below also expose `device_op(dt)`, the `ublr_op_t`
descriptor the CUDA kernels evaluate tiles from, which lets the pipeline
fuse A into the sketch / coupling / near-field kernels (the reference's
matvec ledger still records the columns it would have pushed through A).

* `DenseOperator`: explicit matrix kept in HBM.
* `KernelOperator`: kernel matrices evaluated on the fly (BASELINE configs
  2-5: `-log|x-y|` with diagonal `-log(h/2)`, `1/|x-y|` with diagonal `2/h`).
"""

from __future__ import annotations

import os
from contextlib import contextmanager

import numpy as np

from . import _lib

# ublr_apply_staged for right-hand sides at least this wide on operators at
# least this large (below, the strip evaluation and the GEMM's partial waves
# cost more than evaluating A inside the GEMM saves)
STAGED_MIN_COLS = 512
STAGED_MIN_ROWS = 4096


class LinearOperatorHandle:
    """ref/operators.py:24-35."""

    @property
    def shape(self) -> tuple:
        raise NotImplementedError

    def apply(self, X):
        raise NotImplementedError

    def apply_adjoint(self, X):
        raise NotImplementedError


def _torch():
    import torch
    return torch


def device_apply(inner, perm, x_ptr, ld_x, w, out_ptr, ld_o, device, adjoint=False):
    """out (n x w, ld_o) = A X (ld_x) on the device for an operator with a
    descriptor, rows in the order of `perm`. Kernel operators with a wide
    right-hand side go through ublr_apply_staged (A evaluated once per strip
    of rows into a workspace, then the stored-operand GEMM); everything else
    through ublr_apply (A evaluated inside the GEMM)."""
    torch = _torch()
    desc = inner.device_op(perm, adjoint)
    n = int(desc.n)
    st = _lib.stream_handle()
    if (getattr(inner, "kind", None) in ("log", "inv") and w >= STAGED_MIN_COLS and n >= STAGED_MIN_ROWS
            and os.environ.get("UBLR_APPLY_STAGED", "1") != "0"):
        lib = _lib.load()
        free, _ = torch.cuda.mem_get_info(device)
        nbytes = min(int(lib.ublr_apply_staged_workspace_bytes(n, w)), max(free // 4, 128 * n * 8)) // 8 * 8
        ws = torch.empty(nbytes // 8, dtype=torch.float64, device=device)
        _lib.call("ublr_apply_staged", desc, x_ptr, ld_x, w, out_ptr, ld_o, _lib.ptr(ws), nbytes, st)
        return
    _lib.call("ublr_apply", desc, x_ptr, ld_x, w, out_ptr, ld_o, st)


class _DeviceOperator(LinearOperatorHandle):
    """Common apply/apply_adjoint for operators with a device descriptor.

    Host arrays (original index order) in, host arrays out; CUDA tensors in
    *permuted* (block-contiguous) order are accepted by `apply_device`."""

    symmetric = False

    def _identity_layout(self):
        torch = _torch()
        n = self.shape[0]
        key = "_ident"
        if not hasattr(self, key):
            dev = torch.device("cuda")
            perm = torch.arange(n, dtype=torch.int32, device=dev)
            setattr(self, key, perm)
        return getattr(self, key)

    def apply_device(self, Xd, perm, adjoint=False):
        torch = _torch()
        n, w = Xd.shape
        out = torch.empty((n, w), dtype=torch.float64, device=Xd.device)
        device_apply(self, perm, _lib.ptr(Xd), Xd.stride(0), w, _lib.ptr(out), w, Xd.device, adjoint)
        return out

    def _host_apply(self, X, adjoint):
        torch = _torch()
        _lib.require_device()
        X = np.asarray(X, dtype=float)
        vec = X.ndim == 1
        X2 = X.reshape(-1, 1) if vec else X
        Xd = torch.from_numpy(np.ascontiguousarray(X2)).cuda()
        out = self.apply_device(Xd, self._identity_layout(), adjoint).cpu().numpy()
        return out.ravel() if vec else out

    def apply(self, X):
        return self._host_apply(X, False)

    def apply_adjoint(self, X):
        return self._host_apply(X, not self.symmetric)


class DenseOperator(_DeviceOperator):
    """ref/operators.py:41-52 with the matrix resident in HBM."""

    def __init__(self, matrix):
        torch = _torch()
        if isinstance(matrix, torch.Tensor):
            self.dmatrix = matrix.to(torch.float64).cuda().contiguous()
        else:
            _lib.require_device()
            self.dmatrix = torch.from_numpy(np.ascontiguousarray(matrix, dtype=np.float64)).cuda()
        if self.dmatrix.ndim != 2:
            raise ValueError("DenseOperator needs a 2-D matrix")
        self._shape = tuple(self.dmatrix.shape)

    @property
    def shape(self):
        return self._shape

    @property
    def matrix(self) -> np.ndarray:
        return self.dmatrix.cpu().numpy()

    def device_op(self, perm, adjoint=False):
        d = _lib.OpDesc()
        d.kind = _lib.OP_DENSE
        d.dim = 0
        d.transpose = 1 if adjoint else 0
        d.A = _lib.ptr(self.dmatrix)
        d.lda = self.dmatrix.stride(0)
        d.perm = _lib.ptr(perm)
        d.coords = None
        d.n = self._shape[0]
        d.diag = 0.0
        d._keep = perm
        return d


class KernelOperator(_DeviceOperator):
    """Kernel matrix A(x, y) = f(|x - y|) evaluated on the fly, A(x, x) = diag.

    kind "log": f(r) = -log r (BASELINE configs 2-4, diag -log(h/2));
    kind "inv": f(r) = 1/r (config 5, diag 2/h)."""

    symmetric = True

    def __init__(self, points, kind: str, diag: float):
        coords = np.asarray(getattr(points, "coords", points), dtype=float)
        if coords.ndim != 2 or not 1 <= coords.shape[1] <= 3:
            raise ValueError("coords must be (n, d) with d in 1..3")
        if kind not in ("log", "inv"):
            raise ValueError(f"unknown kernel {kind!r}")
        self.coords = coords
        self.kind = kind
        self.diag = float(diag)
        self._shape = (coords.shape[0], coords.shape[0])
        self._dcoords = {}

    @property
    def shape(self):
        return self._shape

    def _coords_for(self, perm):
        torch = _torch()
        key = perm.data_ptr()
        if key not in self._dcoords:
            p = perm.cpu().numpy()
            soa = np.ascontiguousarray(self.coords[p].T)  # (d, n), permuted
            self._dcoords = {key: (torch.from_numpy(soa).to(perm.device), perm)}
        return self._dcoords[key][0]

    def device_op(self, perm, adjoint=False):
        d = _lib.OpDesc()
        d.kind = _lib.OP_LOG if self.kind == "log" else _lib.OP_INV
        d.dim = self.coords.shape[1]
        d.transpose = 0
        d.A = None
        d.lda = 0
        d.perm = _lib.ptr(perm)
        c = self._coords_for(perm)
        d.coords = _lib.ptr(c)
        d.n = self._shape[0]
        d.diag = self.diag
        d._keep = (perm, c)
        return d

    def dense(self) -> np.ndarray:
        """Materialise A on the host (small problems, tests only)."""
        return self.apply(np.eye(self._shape[0]))


class DifferenceOperator(LinearOperatorHandle):
    """ref/operators.py:55-72."""

    def __init__(self, a, b):
        if a.shape != b.shape:
            raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
        self.a, self.b = a, b

    @property
    def shape(self):
        return self.a.shape

    def apply(self, X):
        return self.a.apply(X) - self.b.apply(X)

    def apply_adjoint(self, X):
        return self.a.apply_adjoint(X) - self.b.apply_adjoint(X)


class MatvecLedger:
    """ref/operators.py:75-125."""

    def __init__(self):
        self.counts = {}
        self._phase = "other"

    @contextmanager
    def phase(self, name: str):
        prev = self._phase
        self._phase = name
        try:
            yield self
        finally:
            self._phase = prev

    def record_apply(self, cols: int):
        self.counts.setdefault(self._phase, [0, 0])[0] += cols

    def record_adjoint(self, cols: int):
        self.counts.setdefault(self._phase, [0, 0])[1] += cols

    def phase_counts(self, name: str) -> tuple:
        a, s = self.counts.get(name, [0, 0])
        return a, s

    def phase_total(self, name: str) -> int:
        return sum(self.counts.get(name, [0, 0]))

    @property
    def count_a(self) -> int:
        return sum(v[0] for v in self.counts.values())

    @property
    def count_astar(self) -> int:
        return sum(v[1] for v in self.counts.values())

    @property
    def total(self) -> int:
        return self.count_a + self.count_astar

    def to_dict(self) -> dict:
        return {name: {"A": v[0], "Astar": v[1]} for name, v in sorted(self.counts.items())}


class CountingOperator(LinearOperatorHandle):
    """ref/operators.py:128-145. Fused GPU paths bill their columns through
    `record_apply` / `record_adjoint` directly."""

    def __init__(self, inner):
        self.inner = inner
        self.ledger = MatvecLedger()

    @property
    def shape(self):
        return self.inner.shape

    def apply(self, X):
        self.ledger.record_apply(X.shape[1] if X.ndim == 2 else 1)
        return self.inner.apply(X)

    def apply_adjoint(self, X):
        self.ledger.record_adjoint(X.shape[1] if X.ndim == 2 else 1)
        return self.inner.apply_adjoint(X)


def counting_wrapper(op) -> CountingOperator:
    return CountingOperator(op)


def unwrap(op):
    while isinstance(op, CountingOperator):
        op = op.inner
    return op
