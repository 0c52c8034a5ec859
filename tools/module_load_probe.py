"""First-launch cost of kernels and kernel modules in a fresh process.

    python tools/module_load_probe.py

Every call is a tiny n=16 run_batch with its layout pinned (SDEB200_LAYOUT, so
no autotune probe runs).  After a warm-up call (context buffers, pinned slots,
the J=2 module) it times: another kernel of an already loaded module, a kernel
of a new module, that kernel again, and a second kernel of that module --
separating per-module from per-function lazy-loading costs.  Run it with
CUDA_MODULE_LOADING=EAGER to compare.
"""

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

t0 = time.perf_counter()
import paper_1908_03869_b200 as sdb  # noqa: E402
from paper_1908_03869_b200 import _native as nat  # noqa: E402

t_import = time.perf_counter() - t0
t0 = time.perf_counter()
nat.context((0,))
t_ctx = time.perf_counter() - t0
batch = sdb.sample_kuramoto_batch(16, 256, (0.2, 0.4), (0.01, 0.1), 0.3, seed=1)
print("import %.1f ms, context %.1f ms (CUDA_MODULE_LOADING=%s)"
      % (1e3 * t_import, 1e3 * t_ctx, os.environ.get("CUDA_MODULE_LOADING", "default")))


def timed(label, lanes, stream):
    os.environ["SDEB200_LAYOUT"] = "%d,0,0,0" % lanes
    cfg = sdb.EngineConfig(dt=1e-3, tspan=2e-3, ksteps=2, orbits=256, lanes=lanes, stream=stream)
    t0 = time.perf_counter()
    sdb.run_batch(sdb.kuramoto_model(16), cfg, batch)
    print("%-44s J=%2d %-12s %.2f ms" % (label, 16 // lanes, stream,
                                         1e3 * (time.perf_counter() - t0)), flush=True)


timed("warm-up (buffers, staging, J=2 module)", 8, "philox")
timed("same module, same kernel", 8, "philox")
timed("same module, another kernel", 8, "sfc64")
timed("new module (J=16)", 1, "philox")
timed("same kernel again", 1, "philox")
timed("same module, another kernel", 1, "sfc64")
timed("same module, a third kernel", 1, "xoshiro256pp")
timed("new module (J=8)", 2, "philox")
timed("new module (J=4)", 4, "philox")
timed("new module (J=1)", 16, "philox")
timed("same module, another kernel", 16, "sfc64")
