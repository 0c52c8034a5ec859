"""SASS of a generated expression-template program (host only, via NVRTC).

    python tools/dsl_sass.py KIND "drift" "diffusion" N NP NN [lanes]
Writes /tmp/dsl_prog.cubin and prints cuobjdump -sass opcode counts.
"""
import ctypes
import os
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1908_03869_b200 import dsl, program  # noqa: E402

kind, drift, diff, n, np_, nn = sys.argv[1:7]
if len(sys.argv) > 7:
    os.environ["SDEB200_DSL_LANES"] = sys.argv[7]
cm = program.compiled(int(n), int(np_), int(nn), dsl.parse(drift), dsl.parse(diff))
src = cm.source(int(kind)).encode()
lib = ctypes.CDLL("/usr/local/cuda/lib64/libnvrtc.so.12")
prog = ctypes.c_void_p()
lib.nvrtcCreateProgram(ctypes.byref(prog), src, b"p.cu", 0, None, None)
opts = [b"-arch=sm_100a", b"-std=c++17", b"--fmad=false", b"-lineinfo",
        ("-I" + os.path.join(ROOT, "paper_1908_03869_b200", "csrc")).encode()]
rc = lib.nvrtcCompileProgram(prog, len(opts), (ctypes.c_char_p * len(opts))(*opts))
sz = ctypes.c_size_t()
lib.nvrtcGetProgramLogSize(prog, ctypes.byref(sz))
log = ctypes.create_string_buffer(sz.value)
lib.nvrtcGetProgramLog(prog, log)
if rc:
    print(log.value.decode())
    sys.exit(1)
lib.nvrtcGetCUBINSize(prog, ctypes.byref(sz))
cubin = ctypes.create_string_buffer(sz.value)
lib.nvrtcGetCUBIN(prog, cubin)
open("/tmp/dsl_prog.cubin", "wb").write(cubin.raw)
sass = subprocess.run(["cuobjdump", "-sass", "/tmp/dsl_prog.cubin"], capture_output=True,
                      text=True).stdout
open("/tmp/dsl_prog.sass", "w").write(sass)
ops = Counter()
for ln in sass.splitlines():
    ln = ln.strip()
    if ln.startswith("/*") and "*/" in ln:
        body = ln.split("*/", 1)[1].strip().rstrip(";").strip()
        if body:
            tok = body.split()
            op = tok[1] if tok[0].startswith("@") else tok[0]
            ops[op.split(".")[0]] += 1
print(sum(ops.values()), "instructions;", ops.most_common(20))
res = subprocess.run(["cuobjdump", "-res-usage", "/tmp/dsl_prog.cubin"], capture_output=True,
                     text=True).stdout
print(res.strip().splitlines()[-1])
