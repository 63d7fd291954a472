"""Build the sm_100a C-ABI library in-tree: paper_2501_05528_b200/libublr_b200.so.

nvcc cross-compiles for B200 without a GPU. Objects go to build/ (git-ignored);
the .so lands next to this file so it travels to the GPU box with the repo.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
GEN = os.path.join(CSRC, "gen")
BUILD = os.path.join(ROOT, "build", "ublr")
LIB = os.path.join(PKG, "libublr_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", f"-I{GEN}", f"-I{os.path.join(ROOT, 'include')}"]
SOURCES = ["capi.cu", "rng.cu", "sketch.cu", "qr.cu", "coupling.cu", "coupling_small.cu", "blr.cu", "dense.cu", "typeb.cu", "tagaspect.cu", "frob.cu", "coupling_gen.cu"]


def _gen_tables():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import gen_ziggurat_tables as g  # noqa: E402
    g.write_header(os.path.join(GEN, "ziggurat_tables.h"))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose):
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    deps.append(os.path.join(ROOT, "include", "ublr_b200.h"))
    if not _stale(obj, deps):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
    with open(obj + ".ptxas.txt", "w") as f:
        f.write(res.stderr)
    return obj, res.stderr if verbose else ""


def build(verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(GEN, exist_ok=True)
    _gen_tables()
    with ThreadPoolExecutor(max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    objs = [o for o, _ in results]
    for _, log in results:
        if log:
            print(log)
    if _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    _build_test_helpers()
    return LIB


def _build_test_helpers():
    """Host-only helper used by the CPU tests to check the RNG decode against
    numpy (tests/native/rng_host.cu). Not part of the product path."""
    src = os.path.join(ROOT, "tests", "native", "rng_host.cu")
    if not os.path.exists(src):
        return
    out = os.path.join(ROOT, "tests", "native", "librng_host.so")
    deps = [src, os.path.join(CSRC, "philox_zig.cuh"), os.path.join(GEN, "ziggurat_tables.h")]
    if not _stale(out, deps):
        return
    cmd = [NVCC, *ARCH, "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", f"-I{GEN}", f"-I{CSRC}", src, "-o", out]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for rng_host.cu:\n{res.stderr}")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
