"""Golden fixtures for the BASELINE configs at their own lengths, made by
running the REFERENCE package itself (build container only: /root/reference).

    python tests/golden/make_golden_r2.py

* cfg1 exactly as BASELINE.json configs[0] states it (n=4, 1,024 orbits,
  dt=1e-3, 10^4 steps, final state) with the reference's Philox stream --
  the complete run_batch, all 1,024 orbits;
* the head rows [0, H) of cfg3 (n = 64, 128, 256 at 1000 / 200 / 100 steps)
  and of the paper's speed protocol (N = 5, 10, 15, dt = 0.05, 8000 steps,
  PAPER.md:228-237): run_batch over speed_protocol_batch(n, H, seed), which
  are exactly the first H rows of the full-size batch (the sampler is keyed
  by orbit id, rng.py:200-222).
The configs mirror bench.py's WORKLOADS (seed 20260809 for both the sampler
and the engine).  Output: golden_r2_v1.npz + cases_r2.json.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("SDEBATCH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from sdebatch import model  # noqa: E402
from sdebatch.engine import EngineConfig, run_batch  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SEED = 20260809
arrays: dict[str, np.ndarray] = {}
cases: dict[str, dict] = {}

# name: (n, head orbits, dt, steps)
RUNS = {
    "cfg1": (4, 1024, 1e-3, 10000),
    "cfg3_n64": (64, 16, 1e-3, 1000),
    "cfg3_n128": (128, 16, 1e-3, 200),
    "cfg3_n256": (256, 8, 1e-3, 100),
    "paper_n5": (5, 32, 0.05, 8000),
    "paper_n10": (10, 32, 0.05, 8000),
    "paper_n15": (15, 32, 0.05, 8000),
}

for name, (n, m, dt, steps) in RUNS.items():
    batch = model.speed_protocol_batch(n, m, SEED)
    cfg = EngineConfig(dt=dt, tspan=dt * steps, ksteps=steps, orbits=m, seed=SEED, threads=1,
                       chunk_group=m)
    t0 = time.perf_counter()
    store = run_batch(model.kuramoto_model(n), cfg, batch)
    wall = time.perf_counter() - t0
    assert not store.failures
    arrays[name + "_init"] = batch.init
    arrays[name + "_params"] = batch.params
    arrays[name + "_values"] = store.values
    cases[name] = {"n": n, "orbits": m, "dt": dt, "steps": steps, "ksteps": steps,
                   "seed": SEED, "stream": "philox", "reference_wall_s": wall}
    print(name, "%.1f s" % wall, flush=True)

np.savez_compressed(os.path.join(HERE, "golden_r2_v1.npz"), **arrays)
with open(os.path.join(HERE, "cases_r2.json"), "w") as f:
    json.dump(cases, f, indent=1)
