"""Build an experimental variant of libsdeb200.so with extra nvcc defines into
its own directory (select it at run time with SDEB200_LIB=<dir>/libsdeb200.so).

    python tools/build_variant.py <name> -DFOO [-DBAR ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1908_03869_b200 import _build as b  # noqa: E402

name, defines = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "paper_1908_03869_b200", "_variants", name)
os.makedirs(out, exist_ok=True)
b.OBJ = os.path.join(out, "obj")
b.LIB = os.path.join(out, "libsdeb200.so")
b.RTC_INC = os.path.join(b.OBJ, "sdeb_rtc_headers.inc")
b.NVCC_FLAGS = [f for f in b.NVCC_FLAGS] + defines
b.NVCC_FLAGS[b.NVCC_FLAGS.index("-I", b.NVCC_FLAGS.index("-I") + 1) + 1] = b.OBJ
print(b.build())
