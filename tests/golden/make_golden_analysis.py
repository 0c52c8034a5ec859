"""Golden fixtures for the analysis row, made by running the
REFERENCE package itself (build container only: /root/reference).

    python tests/golden/make_golden_analysis.py

Records the reference's order_parameter / coherence_series / ensemble_stats /
kymograph_export / wrap_phase on seeded stores, and a small dt_sweep grid
(the accuracy protocol at toy size).  Output: golden_analysis_v1.npz +
cases_analysis.json.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = os.environ.get("SDEBATCH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from sdebatch import analysis, model  # noqa: E402
from sdebatch.engine import EngineConfig, run_batch  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
arrays: dict[str, np.ndarray] = {}
cases: dict[str, dict] = {}

# order parameter of assorted populations (incl. r == 0, huge and negative phases)
g = np.random.default_rng(77)
pops = [np.full(10, 1.3), np.array([0.0, np.pi]), np.array([0.0, np.pi / 2]),
        g.uniform(-50, 50, 17), g.uniform(-np.pi, np.pi, 100), np.array([3.0]),
        g.standard_normal(256) * 1e3, np.array([0.0, 2 * np.pi / 3, 4 * np.pi / 3])]
for k, ph in enumerate(pops):
    pt = analysis.order_parameter(ph)
    arrays["pop_%d" % k] = ph
    arrays["pop_%d_rphi" % k] = np.array([pt.r, pt.phi])
cases["populations"] = len(pops)

# wrap_phase on edge values
w = np.array([-np.pi, np.pi, 0.0, -0.0, 3 * np.pi, -3 * np.pi, 1e9, -7.5, 2 * np.pi, 1e-300])
arrays["wrap_in"] = w
arrays["wrap_out"] = analysis.wrap_phase(w)

# coherence of two Kuramoto runs (one synchronising, one not) + stats + kymograph
for name, (n, m, k_coupling, seed) in {"sync": (16, 12, 0.6, 3), "incoh": (24, 9, 0.01, 4),
                                       "n5": (5, 7, 0.3, 5)}.items():
    cfg = EngineConfig(dt=0.05, tspan=20.0, ksteps=20, orbits=m, seed=seed)
    batch = model.sample_kuramoto_batch(n, m, model.ACCURACY_OMEGA_RANGE,
                                        model.ACCURACY_NOISE_RANGE, k_coupling, seed)
    store = run_batch(model.kuramoto_model(n), cfg, batch)
    cs = analysis.coherence_series(store)
    st = analysis.ensemble_stats(cs)
    arrays[name + "_init"] = batch.init
    arrays[name + "_params"] = batch.params
    arrays[name + "_values"] = store.values
    arrays[name + "_r"] = cs.r
    arrays[name + "_phi"] = cs.phi
    arrays[name + "_mean_r"] = st.mean_r
    arrays[name + "_std_r"] = st.std_r
    arrays[name + "_kymo1"] = analysis.kymograph_export(store, 1)
    cases[name] = dict(n=n, orbits=m, coupling=k_coupling, seed=seed, dt=0.05, tspan=20.0,
                       ksteps=20,
                       first_cross=analysis.first_crossing_time(cs.times, st.mean_r, 0.5))

# a toy dt sweep (the accuracy protocol: couplings x dts, realizations)
rows = analysis.dt_sweep(6, couplings=[0.02, 0.2], dts=[0.05, 0.1], realizations=8,
                         tspan=4.0, sample_interval=0.5, seed=21, threads=1)
cases["dt_sweep"] = [dict(coupling=r.coupling, dt=r.dt, mean_r_end=r.mean_r_end,
                          std_r_end=r.std_r_end) for r in rows]
for k, r in enumerate(rows):
    arrays["sweep_%d_mean" % k] = r.stats.mean_r
    arrays["sweep_%d_std" % k] = r.stats.std_r
    arrays["sweep_%d_times" % k] = r.stats.times

np.savez_compressed(os.path.join(HERE, "golden_analysis_v1.npz"), **arrays)
with open(os.path.join(HERE, "cases_analysis.json"), "w") as f:
    json.dump(cases, f, indent=1, sort_keys=True)
print("wrote %d arrays" % len(arrays))
