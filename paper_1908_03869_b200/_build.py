"""Builds libsdeb200.so in-tree with nvcc for sm_100a (no JIT, no torch build).

``python -m paper_1908_03869_b200._build`` or ``__graft_entry__.build()``.
Objects compile in parallel; the shared library links cudart statically so
it loads (and exports every include/sdeb200.h symbol) on a machine without a
GPU, which the CPU test tier checks.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libsdeb200.so")

SOURCES = ["sdeb_capi.cu", "sdeb_misc.cu"] + ["sdeb_kuramoto_j%d.cu" % j for j in (1, 2, 4, 8, 16)]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: every FP64 op on the stepper path is an explicit __d*_rn /
# __fma_rn intrinsic already; the flag pins the rest (libdevice's huge-argument
# trig reduction multiplies by 2/pi with a plain `*`), which ptxas would
# otherwise fuse differently per kernel instantiation -- breaking the
# bit-identity of lane layouts for |theta| >= 2^29.
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libsdeb200.so")


def _mtime(path: str) -> float:
    return os.path.getmtime(path) if os.path.exists(path) else -1.0


def _compile(src: str, log: list) -> str:
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS]
    deps.append(os.path.join(ROOT, "include", "sdeb200.h"))
    if _mtime(obj) >= max(_mtime(d) for d in deps):
        return obj
    cmd = [nvcc()] + NVCC_FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log.append((src, res.stdout + res.stderr))
    if res.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s" % (src, res.stdout + res.stderr))
    return obj


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in os.listdir(OBJ):
            os.remove(os.path.join(OBJ, f))
    log: list = []
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        objs = list(pool.map(lambda s: _compile(s, log), SOURCES))
    if force or _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("link failed:\n" + res.stdout + res.stderr)
    if verbose:
        for src, text in log:
            sys.stdout.write("== %s\n%s" % (src, text))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="--force" in sys.argv))
