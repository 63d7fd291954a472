"""ctypes binding of the C-ABI library libublr_b200.so (include/ublr_b200.h).

The product path has no CPU fallback: if the library is missing or no sm_100
device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libublr_b200.so")

UBLR_OK, UBLR_ERR_VALUE, UBLR_ERR_CUDA, UBLR_ERR_NUMERIC = 0, -1, -2, -3
OP_DENSE, OP_LOG, OP_INV = 0, 1, 2

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
INT = C.c_int


class OpDesc(C.Structure):
    _fields_ = [("kind", I32), ("dim", I32), ("transpose", I32), ("pad_", I32),
                ("A", P), ("lda", I64), ("perm", P), ("coords", P), ("n", I64), ("diag", C.c_double)]


class RngStreamDesc(C.Structure):
    _fields_ = [("key0", C.c_uint64), ("key1", C.c_uint64), ("count", I64), ("cols", I64),
                ("ld", I64), ("out_offset", I64), ("rowmap", P)]


RNG_STREAM_DTYPE = np.dtype([("key0", "<u8"), ("key1", "<u8"), ("count", "<i8"), ("cols", "<i8"),
                             ("ld", "<i8"), ("out_offset", "<i8"), ("rowmap", "<u8")])
assert RNG_STREAM_DTYPE.itemsize == C.sizeof(RngStreamDesc)

# name -> (restype, argtypes); must cover every function in include/ublr_b200.h
SIGNATURES = {
    "ublr_last_error": (C.c_char_p, []),
    "ublr_version": (INT, []),
    "ublr_device_check": (INT, []),
    "ublr_seedseq_keys": (INT, [P, INT, P, INT, P, INT, I64, P]),
    "ublr_null_vectors": (INT, [P, INT, P, P, INT, P, P]),
    "ublr_tag_plan_host": (INT, [P, INT, P, P, INT, P, P, P, P]),
    "ublr_tag_aspect": (INT, [P, P, INT, P, P, INT, P, P]),
    "ublr_null_vectors_device": (INT, [P, INT, P, P, INT, P, P, P]),
    "ublr_rng_workspace_bytes": (I64, [P, INT]),
    "ublr_rng_normals": (INT, [P, P, INT, P, P, I64, P]),
    "ublr_sketch_tagged": (INT, [C.POINTER(OpDesc), P, INT, P, INT, P, I64, INT, P, I64, INT, INT, P]),
    "ublr_sketch_tagged_pair": (INT, [C.POINTER(OpDesc), P, INT, P, INT, P, P, I64, INT, P, P, I64, INT, INT, P]),
    "ublr_sketch_tagged_comp": (INT, [C.POINTER(OpDesc), P, INT, P, INT, P, P, I64, INT, P, P, I64, INT, INT, P]),
    "ublr_sketch_tagged_staged": (INT, [C.POINTER(OpDesc), P, INT, P, INT, P, P, I64, INT, P, P, I64, INT, INT, INT,
                                        P, I64, P]),
    "ublr_sketch_tagged_staged_rows": (INT, [I64, INT, INT, I64]),
    "ublr_sketch_tagged_two": (INT, [C.POINTER(OpDesc), C.POINTER(OpDesc), P, INT, P, INT, P, P, I64, INT, P, P, I64,
                                     INT, INT, P]),
    "ublr_apply": (INT, [C.POINTER(OpDesc), P, I64, INT, P, I64, P]),
    "ublr_apply_staged": (INT, [C.POINTER(OpDesc), P, I64, INT, P, I64, P, I64, P]),
    "ublr_apply_staged_workspace_bytes": (I64, [I64, INT]),
    "ublr_apply_staged_rows": (INT, [I64, INT, I64]),
    "ublr_block_qr": (INT, [P, I64, INT, P, INT, INT, P, P, INT, INT, P, I64, P, INT]),
    "ublr_block_qr_pair": (INT, [P, P, I64, P, INT, INT, P, INT, INT, P, P, I64, P, INT]),
    "ublr_coupling": (INT, [C.POINTER(OpDesc), P, P, INT, INT, P, P, I64, P, I64, P, INT, INT, INT]),
    "ublr_nearfield_workspace_bytes": (I64, [INT, INT, INT]),
    "ublr_coupling_nearfield": (INT, [C.POINTER(OpDesc), P, P, INT, INT, P, P, I64, P, I64, P, P, INT, INT, P, P, P,
                                      P, P, INT, INT]),
    "ublr_blr_apply_workspace_bytes": (I64, [I64, INT]),
    "ublr_gemm_batched": (INT, [INT, INT, INT, INT, INT, C.c_double, P, I64, I64, P, I64, P, I64, I64, P, I64,
                                C.c_double, P, I64, I64, P, I64, INT, P]),
    "ublr_potrf_diag": (INT, [P, I64, I64, INT, INT, P, I64, I64, P, P, INT, P]),
    "ublr_lu_sign_diag": (INT, [P, I64, I64, INT, INT, P, I64, I64, P, P, P, I64, P, INT, P]),
    "ublr_lu_sign_diag_r": (INT, [P, I64, I64, INT, INT, P, I64, I64, P, P, P, I64, P, P, I64, I64, INT, INT, P]),
    "ublr_syrk_upper_batched": (INT, [INT, INT, C.c_double, P, I64, I64, C.c_double, P, I64, I64, INT, P]),
    "ublr_add_scaled_rows": (INT, [P, I64, I64, P, I64, I64, P, I64, INT, INT, INT, P]),
    "ublr_gather": (INT, [P, I64, I64, P, I64, INT, INT, INT, INT, P, I64, I64, INT, P]),
    "ublr_scale_rows": (INT, [P, I64, I64, P, I64, INT, INT, INT, P]),
    "ublr_assemble_gram": (INT, [P, P, INT, INT, P, INT, P]),
    "ublr_tag_combine_pairs": (INT, [P, I64, INT, INT, P, P, P, INT, INT, P, P]),
    "ublr_pairs_pad": (INT, [P, P, P, P, P, INT, INT, P, INT, P]),
    "ublr_assemble_tagged": (INT, [P, INT, P, I64, INT, P, INT, P, I64, I64, P]),
    "ublr_blr_apply": (INT, [P, P, I64, P, I64, P, P, P, P, P, P, P, INT, P, I64, INT, INT, P, I64, P, P]),
    "ublr_frob_error": (INT, [C.POINTER(OpDesc), P, P, P, P, INT, P, INT, P, P, I64, P, I64, P, INT, INT, P, P, P]),
    "ublr_frob_diff": (INT, [P, P, P, P, INT, P, INT, P, P, I64, P, I64, P, P, INT, P, P, I64, P, I64, P, INT, INT, P,
                             P]),
    "ublr_nearfield_colour": (INT, [C.POINTER(OpDesc), P, P, INT, INT, P, P, I64, P, I64, P, P, P, INT, INT,
                                    P, P, INT, P, P, P, I64, P]),
}

_lib = None


def load():
    """Load the library (no GPU needed); raise ImportError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2501_05528_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class UblrCudaError(RuntimeError):
    pass


def check(rc: int, what: str = ""):
    if rc == UBLR_OK:
        return
    msg = load().ublr_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == UBLR_ERR_VALUE:
        raise ValueError(text)
    if rc == UBLR_ERR_NUMERIC:
        raise np.linalg.LinAlgError(text)
    raise UblrCudaError(text)


# kernels each C-ABI entry point launches (for bench.py's `gpu_launches`)
LAUNCHES = {"ublr_rng_normals": 8, "ublr_sketch_tagged": 1, "ublr_sketch_tagged_pair": 1, "ublr_sketch_tagged_comp": 1, "ublr_sketch_tagged_two": 1, "ublr_apply": 1,
            "ublr_block_qr": 1, "ublr_block_qr_pair": 1, "ublr_coupling": 1, "ublr_nearfield_colour": 2,
            "ublr_coupling_nearfield": 1,
            "ublr_blr_apply": 3, "ublr_gemm_batched": 1, "ublr_potrf_diag": 1, "ublr_lu_sign_diag": 1,
            "ublr_lu_sign_diag_r": 1, "ublr_syrk_upper_batched": 1, "ublr_add_scaled_rows": 1,
            "ublr_gather": 1, "ublr_scale_rows": 1, "ublr_tag_combine_pairs": 1, "ublr_assemble_tagged": 1, "ublr_tag_aspect": 1, "ublr_null_vectors_device": 1,
            "ublr_frob_error": 1, "ublr_frob_diff": 1, "ublr_pairs_pad": 1}
launch_count = 0


def rng_launches(counts) -> int:
    """Kernels one ublr_rng_normals call launches (rng.cu: one per-CTA decode
    kernel for short streams, else the 8-kernel chunk-parallel set)."""
    path = os.environ.get("UBLR_RNG_PATH", "0")
    mx = int(np.max(counts)) if len(counts) else 0
    if path == "2" or (path == "0" and (mx + mx // 24 + 256 + 15) // 16 <= 512):
        return 1
    return LAUNCHES["ublr_rng_normals"]


def _launches_of(name, args):
    if name == "ublr_sketch_tagged_staged":   # one evaluation + one sketch launch per strip of rows
        n, gc, r0, r1, nbytes = int(args[0].n), int(args[8]), int(args[12]), int(args[13]), int(args[16])
        rows = int(load().ublr_sketch_tagged_staged_rows(n, (2 if args[6] else 1) * gc, r1 - r0, nbytes))
        return 2 * -(-(r1 - r0) // rows) if rows >= 32 else 2
    if name == "ublr_apply_staged":   # one evaluation + one GEMM launch per strip of rows
        n, w, nbytes = int(args[0].n), int(args[3]), int(args[7])
        rows = max(128, int(load().ublr_apply_staged_rows(n, w, nbytes)))
        return 2 * -(-n // rows)
    return LAUNCHES.get(name, 0)
_events = None  # name -> list of (start, end) CUDA events when instrumentation is on


work = {}  # name -> algorithmic flops issued while instrumenting


def add_work(name: str, flops: float):
    """Algorithmic flop count of a launch (bench.py roofline numerator)."""
    if _events is not None:
        work[name] = work.get(name, 0.0) + float(flops)


_only = None  # instrument only these entry points (None: all)


def instrument(enable: bool = True, only=None):
    """Record CUDA events around C-ABI launches (bench.py roofline): every
    entry point, or just the names in `only` (two event records per launch
    of host time, so the timed bench region instruments only the kernel it
    reports)."""
    global _events, _only
    _events = {} if enable else None
    _only = set(only) if only else None
    if enable:
        work.clear()


def event_times():
    """{name: [ms per call]} of the instrumented calls (synchronises)."""
    import torch
    torch.cuda.synchronize()
    return {k: [a.elapsed_time(b) for a, b in v] for k, v in (_events or {}).items()}


def _work_of(name, args):
    """Algorithmic fp64 flops of the hot entry points, from their arguments."""
    try:
        if name in ("ublr_apply", "ublr_apply_staged"):
            n = args[0].n
            return 2.0 * n * n * int(args[3])
        if name == "ublr_sketch_tagged_two":
            n, b, ell, gc = args[0].n, int(args[3]), int(args[5]), int(args[9])
            r0, r1 = int(args[13]), int(args[14])
            return 2 * (2.0 * (r1 - r0) * n * gc + 2.0 * (r1 - r0) * b * gc * ell)
        if name in ("ublr_sketch_tagged", "ublr_sketch_tagged_pair", "ublr_sketch_tagged_comp",
                    "ublr_sketch_tagged_staged"):
            pair = not name.endswith("tagged")
            n, b, ell = args[0].n, int(args[2]), int(args[4])
            gc = int(args[8] if pair else args[7])
            r0, r1 = (int(args[12]), int(args[13])) if pair else (int(args[10]), int(args[11]))
            cols = (2 if pair and args[6] else 1) * gc
            return 2.0 * (r1 - r0) * n * cols + 2.0 * (r1 - r0) * b * cols * ell
        if name == "ublr_gemm_batched":
            return 2.0 * int(args[2]) * int(args[3]) * int(args[4]) * int(args[22])
        if name == "ublr_syrk_upper_batched":
            return 1.0 * int(args[0]) * (int(args[0]) + 1) * int(args[1]) * int(args[10])
        if name == "ublr_coupling":
            n, b, k, m = args[0].n, int(args[3]), int(args[4]), int(args[11])
            rows = (int(args[13]) - int(args[12])) * m
            return 2.0 * rows * n * k + 2.0 * rows * (b * k) * k
        if name == "ublr_coupling_nearfield":
            n, b, k, m = args[0].n, int(args[3]), int(args[4]), int(args[13])
            rows = (int(args[20]) - int(args[19])) * m
            return 2.0 * rows * n * k + 2.0 * rows * (b * k) * k
    except Exception:  # pragma: no cover - accounting only
        return 0.0
    return 0.0


def call(name: str, *args, launches=None, on=None):
    """Call a status-returning C-ABI function and raise on failure
    (`launches`: kernels it launches when that depends on the arguments;
    `on`: the torch stream it launches on when that is not the current one,
    for the instrumentation events)."""
    global launch_count
    launch_count += _launches_of(name, args) if launches is None else launches
    if _events is not None and (_only is None or name in _only):
        add_work(name, _work_of(name, args))
        import torch
        st = current_stream() if on is None else on
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        check(getattr(load(), name)(*args), name)
        b.record(st)
        _events.setdefault(name, []).append((a, b))
        return
    check(getattr(load(), name)(*args), name)


_device_ok = False


def require_device():
    """The CUDA path is the only path: fail loudly without an sm_100 GPU."""
    global _device_ok
    if _device_ok:
        return
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2501_05528_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")
    torch.cuda.init()
    call("ublr_device_check")
    _device_ok = True


def ptr(t) -> int:
    """Device pointer of a torch tensor (0 for None; ints pass through)."""
    if t is None:
        return 0
    if isinstance(t, int):    # already a raw device address
        return t
    return int(t.data_ptr())


class _PinnedRing:
    """Small host->device transfers staged through a ring of pinned slots.
    A slot is reused only after the copy that last read it has completed
    (its CUDA event), so the caller never blocks on the GPU in practice and a
    pageable copy (which would wait for all queued work) is never issued."""

    SLOT = 1 << 20
    NSLOT = 16

    def __init__(self):
        import torch
        self.buf = torch.empty(self.SLOT * self.NSLOT, dtype=torch.uint8, pin_memory=True)
        self.np = self.buf.numpy()
        self.events = [torch.cuda.Event() for _ in range(self.NSLOT)]
        self.used = [False] * self.NSLOT
        self.i = 0

    def h2d(self, a, device):
        import torch
        a = np.ascontiguousarray(a)
        nb = a.nbytes
        if nb > self.SLOT or nb == 0:
            t = torch.from_numpy(a)
            return t.pin_memory().to(device, non_blocking=True) if nb else t.to(device)
        s = self.i
        self.i = (self.i + 1) % self.NSLOT
        if self.used[s]:
            self.events[s].synchronize()
        off = s * self.SLOT
        view = self.np[off:off + nb].view(a.dtype).reshape(a.shape)
        view[...] = a
        out = torch.from_numpy(view).to(device, non_blocking=True)
        self.events[s].record(current_stream())
        self.used[s] = True
        return out


_ring = None


def h2d(a, device):
    """Host array -> device tensor without blocking the host (pinned staging
    ring, non_blocking copy on the current stream)."""
    global _ring
    if _ring is None:
        _ring = _PinnedRing()
    return _ring.h2d(a, device)


_stream_cached = None


class stream_scope:
    """Within the scope, stream_handle() returns the current stream captured
    at entry (torch.cuda.current_stream() costs ~10 us per call; a compression
    issues dozens of launches on one stream)."""

    def __enter__(self):
        global _stream_cached, _stream_obj
        import torch
        self._prev = (_stream_cached, _stream_obj)
        # the raw handle is a cheap query; the torch Stream object (for
        # Event.record) is memoised per (device, handle)
        dev = torch._C._cuda_getDevice()
        raw = torch._C._cuda_getCurrentRawStream(dev)
        hit = _STREAMS.get((dev, raw))
        if hit is None:
            obj = torch.cuda.current_stream()
            if len(_STREAMS) > 64:
                _STREAMS.clear()
            hit = _STREAMS[(dev, raw)] = (obj, C.c_void_p(raw))
        _stream_obj, _stream_cached = hit
        return self

    def __exit__(self, *exc):
        global _stream_cached, _stream_obj
        _stream_cached, _stream_obj = self._prev


_stream_obj = None
_STREAMS = {}   # (device, raw handle) -> (torch Stream, c_void_p)
_SIDE = {}      # (device, main raw handle) -> (torch Stream, c_void_p)


def side_stream():
    """A second stream for work that is independent of the kernel queued
    next on the current one (one per device and current stream, created
    once): (torch Stream, raw handle)."""
    import torch
    main = current_stream()
    key = (main.device_index, main.cuda_stream)
    hit = _SIDE.get(key)
    if hit is None:
        st = torch.cuda.Stream(device=main.device)
        hit = _SIDE[key] = (st, C.c_void_p(st.cuda_stream))
    return hit


def current_stream():
    """torch.cuda.current_stream(), cached inside a stream_scope (pass it to
    Event.record: without an argument, record() queries the current stream)."""
    if _stream_obj is not None:
        return _stream_obj
    import torch
    return torch.cuda.current_stream()


def stream_handle():
    if _stream_cached is not None:
        return _stream_cached
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)
