"""First-launch cost per kernel module in a fresh process.

    python tools/module_load_probe.py            # CUDA_MODULE_LOADING as set

For each lane width J (each J is its own kernel module, sdeb_kuramoto_j*.cu)
times the first and the second run_batch of a tiny n=16 run pinned to that
layout.  The difference is what a cold call pays for loading the module the
layout lives in.
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
for lanes in (1, 2, 4, 8, 16):
    cfg = sdb.EngineConfig(dt=1e-3, tspan=2e-3, ksteps=2, orbits=256, lanes=lanes)
    times = []
    for _ in range(2):
        t0 = time.perf_counter()
        sdb.run_batch(sdb.kuramoto_model(16), cfg, batch)
        times.append(1e3 * (time.perf_counter() - t0))
    print("J=%2d: first %.2f ms, second %.2f ms" % (16 // lanes, times[0], times[1]), flush=True)
