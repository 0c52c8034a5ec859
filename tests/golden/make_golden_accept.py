"""Golden fixture for the reference's acceptance criteria 1-3, made by
running the REFERENCE package itself (build container only: /root/reference).

    python tests/golden/make_golden_accept.py

Runs the reference's own synchronisation-transition sweep exactly as its
acceptance suite does (test_acceptance.py:36-42: analysis.dt_sweep(100,
couplings=(0.02, 0.2), dts=STABILITY_DT_VALUES, realizations=64, tspan=400,
sample_interval=2, seed=20260809)) and records every row's ensemble mean and
std of r over time.  Output: golden_accept_v1.npz (+ the wall time in
cases_accept.json).  Takes ~10-15 min on 8 cores.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("SDEBATCH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from sdebatch import analysis  # noqa: E402
from sdebatch.analysis import STABILITY_DT_VALUES  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ACCEPT_SEED = 20260809
SWEEP_COUPLINGS = (0.02, 0.2)

t0 = time.perf_counter()
rows = analysis.dt_sweep(100, couplings=SWEEP_COUPLINGS, dts=STABILITY_DT_VALUES,
                         realizations=64, tspan=400.0, sample_interval=2.0, seed=ACCEPT_SEED,
                         threads="all")
wall = time.perf_counter() - t0
arrays = {"couplings": np.array([r.coupling for r in rows]),
          "dts": np.array([r.dt for r in rows]),
          "mean_r_end": np.array([r.mean_r_end for r in rows]),
          "std_r_end": np.array([r.std_r_end for r in rows]),
          "times": rows[0].stats.times,
          "mean_r": np.stack([r.stats.mean_r for r in rows]),
          "std_r": np.stack([r.stats.std_r for r in rows])}
np.savez_compressed(os.path.join(HERE, "golden_accept_v1.npz"), **arrays)
with open(os.path.join(HERE, "cases_accept.json"), "w") as f:
    json.dump({"seed": ACCEPT_SEED, "couplings": list(SWEEP_COUPLINGS),
               "dts": list(STABILITY_DT_VALUES), "realizations": 64, "tspan": 400.0,
               "sample_interval": 2.0, "n": 100, "reference_wall_s": wall,
               "source": "sdebatch.analysis.dt_sweep (reference, unmodified)"}, f, indent=1)
print("rows", len(rows), "wall %.1f s" % wall)
for r in rows:
    print(r.coupling, r.dt, r.mean_r_end, r.std_r_end)
