"""Builds libsdeb200.so in-tree with nvcc for sm_100a (no JIT, no torch build).

``python -m paper_1908_03869_b200._build`` or ``__graft_entry__.build()``.
Objects compile in parallel and are rebuilt when their content key changes
(sha256 of the source, every header, the flags and nvcc's version; stored
next to each object as ``<obj>.key``).  The shared library links cudart statically so
it loads (and exports every include/sdeb200.h symbol) on a machine without a
GPU, which the CPU test tier checks.
"""

from __future__ import annotations

import hashlib
import os
import re
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libsdeb200.so")

# stepper instantiations: power-of-two lane widths J, plus every other J <= 16
# for the exact one-lane layouts of n = J (sdeb_capi.cu exact_J)
EXACT_J = (3, 5, 6, 7, 9, 10, 11, 12, 13, 14, 15)
SOURCES = (["sdeb_capi.cu", "sdeb_misc.cu", "sdeb_dsl.cu"]
           + ["sdeb_kuramoto_j%d.cu" % j for j in (1, 2, 4, 8, 16) + EXACT_J])
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))
# device headers the NVRTC-compiled expression-template programs include; they
# are embedded into the library (no source tree needed at run time)
RTC_HEADERS = ["sdeb_dsl_kernel.cuh", "sdeb_dsl_args.h", "sdeb_rng.cuh", "sdeb_math.cuh",
               "sdeb_cstdint.cuh", "sdeb_log_table.cuh", "sdeb_sincos_table.cuh"]
RTC_INC = os.path.join(OBJ, "sdeb_rtc_headers.inc")
CUDA_LIB = "/usr/local/cuda/lib64"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: every FP64 op on the stepper path is an explicit __d*_rn /
# __fma_rn intrinsic already; the flag pins the rest (libdevice's huge-argument
# trig reduction multiplies by 2/pi with a plain `*`), which ptxas would
# otherwise fuse differently per kernel instantiation -- breaking the
# bit-identity of lane layouts for |theta| >= 2^29.
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), "-I", OBJ]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libsdeb200.so")


def _mtime(path: str) -> float:
    return os.path.getmtime(path) if os.path.exists(path) else -1.0


_TOOLCHAIN = None


def toolchain_id() -> str:
    """nvcc's version banner: part of every build key, so a different toolkit
    rebuilds everything."""
    global _TOOLCHAIN
    if _TOOLCHAIN is None:
        res = subprocess.run([nvcc(), "--version"], capture_output=True, text=True)
        _TOOLCHAIN = res.stdout.strip()
    return _TOOLCHAIN


def _digest(*parts) -> str:
    h = hashlib.sha256()
    for part in parts:
        if isinstance(part, str) and os.path.isfile(part):
            with open(part, "rb") as f:
                h.update(f.read())
        else:
            h.update(repr(part).encode())
        h.update(b"\0")
    return h.hexdigest()


def _stamp_ok(target: str, key: str) -> bool:
    """The target exists and was built from exactly this key (content hash of
    sources, headers, flags and toolchain -- not modification times, which do
    not survive a copy of the tree)."""
    try:
        with open(target + ".key") as f:
            return os.path.exists(target) and f.read().strip() == key
    except OSError:
        return False


def _write_stamp(target: str, key: str) -> None:
    with open(target + ".key", "w") as f:
        f.write(key + "\n")


def _write_rtc_headers() -> None:
    """sdeb_rtc_headers.inc: {name, raw text} of every header a generated
    program includes (rewritten only when its content changes)."""
    parts = ["const RtcHeader kRtcHeaders[] = {"]
    for h in RTC_HEADERS:
        with open(os.path.join(CSRC, h)) as f:
            text = f.read()
        assert ")SDEBRTC\"" not in text
        # split into <= 60 KB raw-string pieces (adjacent literals concatenate)
        chunks = [text[i:i + 60000] for i in range(0, len(text), 60000)] or [""]
        body = "\n".join('R"SDEBRTC(%s)SDEBRTC"' % c for c in chunks)
        parts.append('    {"%s",\n%s},' % (h, body))
    parts.append("};")
    text = "\n".join(parts) + "\n"
    if os.path.exists(RTC_INC):
        with open(RTC_INC) as f:
            if f.read() == text:
                return
    tmp = RTC_INC + ".tmp"
    with open(tmp, "w") as f:
        f.write(text)
    os.replace(tmp, RTC_INC)


def _compile(src: str, log: list) -> str:
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS]
    if src == "sdeb_dsl.cu":
        deps.append(RTC_INC)
    if src == "sdeb_capi.cu":
        deps.append(KERNEL_TABLE)
    deps.append(os.path.join(ROOT, "include", "sdeb200.h"))
    key = _digest(toolchain_id(), NVCC_FLAGS, src, *deps)
    if _stamp_ok(obj, key) and os.path.exists(obj + ".ptxas"):
        return obj
    cmd = [nvcc()] + NVCC_FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log.append((src, res.stdout + res.stderr))
    if res.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s" % (src, res.stdout + res.stderr))
    with open(obj + ".ptxas", "w") as f:  # resource usage, read by _write_kernel_table
        f.write(res.stdout + res.stderr)
    _write_stamp(obj, key)
    return obj


KERNEL_TABLE = os.path.join(OBJ, "sdeb_kernel_table.inc")
_ENTRY = re.compile(r"Compiling entry function '_ZN4sdeb19kuramoto_run_kernelILi(\d+)ELi(\d+)"
                    r"ELi(\d+)ELi(\d+)ELi(\d+)EEEvNS_7RunArgsE'")
_USED = re.compile(r"Used (\d+) registers.*?(\d+) bytes smem")


def _write_kernel_table(objs) -> None:
    """sdeb_kernel_table.inc: registers and static shared memory of every
    kuramoto_run_kernel instantiation, from ptxas -v of the stepper objects.
    The layout autotuner estimates occupancy from it without touching (and so
    lazily loading) kernel modules it may never launch."""
    rows = set()
    for obj in objs:
        try:
            with open(obj + ".ptxas") as f:
                text = f.read()
        except OSError:
            continue
        cur = None
        for ln in text.splitlines():
            m = _ENTRY.search(ln)
            if m:
                cur = tuple(int(x) for x in m.groups())
                continue
            m = _USED.search(ln)
            if m and cur:
                rows.add(cur + (int(m.group(1)), int(m.group(2))))
                cur = None
    body = ["// generated by _build.py from ptxas -v; {J, solver, stream, coupling, variant, "
            "registers, static smem bytes}",
            "const KernelRes kKernelRes[] = {"]
    body += ["    {%d, %d, %d, %d, %d, %d, %d}," % r for r in sorted(rows)]
    body += ["    {0, 0, 0, 0, 0, 0, 0},", "};", ""]
    text = "\n".join(body)
    if os.path.exists(KERNEL_TABLE):
        with open(KERNEL_TABLE) as f:
            if f.read() == text:
                return
    with open(KERNEL_TABLE + ".tmp", "w") as f:
        f.write(text)
    os.replace(KERNEL_TABLE + ".tmp", KERNEL_TABLE)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in os.listdir(OBJ):
            os.remove(os.path.join(OBJ, f))
    _write_rtc_headers()
    log: list = []
    # the stepper objects first: their ptxas resource usage becomes a table the
    # host code (sdeb_capi.cu) is compiled with
    steppers = [x for x in SOURCES if x.startswith("sdeb_kuramoto_j")]
    others = [x for x in SOURCES if x not in steppers]
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        stepper_objs = list(pool.map(lambda s: _compile(s, log), steppers))
        _write_kernel_table(stepper_objs)
        objs = list(pool.map(lambda s: _compile(s, log), others)) + stepper_objs
    cmd = ([nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs
           + ["-L", CUDA_LIB, "-lnvrtc", "-Xlinker", "-rpath=" + CUDA_LIB])
    lib_key = _digest(toolchain_id(), cmd, *objs)
    if force or not _stamp_ok(LIB, lib_key):
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("link failed:\n" + res.stdout + res.stderr)
        _write_stamp(LIB, lib_key)
    if verbose:
        for src, text in log:
            sys.stdout.write("== %s\n%s" % (src, text))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="--force" in sys.argv))
