"""In-tree build of libdsfft.so (sm_100a) -- ``python -m paper_2604_00567_b200.build``.

Compiles every CUDA translation unit with
``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` (one object per
transform size so the unrolled kernels build in parallel), the host table
builder with g++ ``-ffp-contract=off`` (the reference's rule), and links
``paper_2604_00567_b200/libdsfft.so`` next to this file, where the ctypes
loader finds it.  Incremental: objects newer than their sources are reused.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libdsfft.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xcompiler", "-ffp-contract=off", f"-I{ROOT}/include", f"-I{CSRC}"]
SMALL_SIZES = range(1, 14)


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def _stale(obj, srcs):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(s) > t for s in srcs)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stderr


def jobs():
    hdr = _headers()
    out = []
    for m in SMALL_SIZES:
        src = os.path.join(CSRC, "inst_small.cu")
        obj = os.path.join(OBJ, f"inst_m{m}.o")
        out.append((obj, [src] + hdr, [NVCC] + NVFLAGS + [f"-DDSFFT_M={m}", "-c", src, "-o", obj]))
    for name in ("dsfft_capi.cu", "multipass.cu", "multipass_fused.cu", "fp64.cu", "error_harness.cu",
                 "synth.cu", "emulate.cu"):
        src = os.path.join(CSRC, name)
        obj = os.path.join(OBJ, name.replace(".cu", ".o"))
        out.append((obj, [src] + hdr, [NVCC] + NVFLAGS + ["-c", src, "-o", obj]))
    src = os.path.join(CSRC, "host_table.cpp")
    obj = os.path.join(OBJ, "host_table.o")
    out.append((obj, [src] + hdr, ["g++", "-O2", "-fPIC", "-std=c++17", "-ffp-contract=off",
                                   "-Wall", "-Wextra", f"-I{CSRC}", "-c", src, "-o", obj]))
    return out


def build(verbose: bool = False, workers: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    todo = [(o, c) for o, srcs, c in jobs() if _stale(o, srcs)]
    workers = workers or min(len(todo) or 1, os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(workers) as ex:
        for (o, c), log in zip(todo, ex.map(lambda oc: _run(oc[1]), todo)):
            if verbose:
                print("built", os.path.relpath(o, ROOT), file=sys.stderr)
                if log.strip():
                    print(log, file=sys.stderr)
    objs = [o for o, _, _ in jobs()]
    if _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lpthread"])
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
