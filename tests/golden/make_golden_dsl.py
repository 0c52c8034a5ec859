"""Golden fixtures for expression-template models, made by running the
REFERENCE package itself (build container only: /root/reference).

    python tests/golden/make_golden_dsl.py

Records, for small seeded inputs, ``run_batch`` stores of models built with
the reference's ``model_from_dsl`` (em / euler / rk4, time dependence, powers,
nested sums, every function, failures, a system above the unroll limit) plus
``drift_eval`` / ``diffusion_eval`` values.  Output: golden_dsl_v1.npz +
cases_dsl.json (committed; read by tests on any machine).
"""

from __future__ import annotations

import json
import zlib
import os
import sys

import numpy as np

REF = os.environ.get("SDEBATCH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from sdebatch import model  # noqa: E402
from sdebatch.engine import EngineConfig, run_batch  # noqa: E402
from sdebatch.model import OrbitBatch  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# name: (nequat, nparams, nnoise, drift, diffusion, solver, orbits, dt, steps, ksteps, seed)
MODELS = {
    "ou": (3, 5, 3, "p[0]*(p[1] - y[i])", "p[2 + i]*n[i]", "em", 16, 0.01, 200, 20, 11),
    "tdep": (4, 8, 4, "-(y[i]^3) + sin(t)*p[i] + cos(2*t)*y[i]/N",
             "p[N + i] * n[i] * sqrt(1 + y[i]^2)", "em", 12, 0.005, 240, 40, 7),
    "nested": (3, 9, 3, "sum(j, sum(k, p[3*j + k] * sin(y[k] - y[j]))) / N^2 - 0.1*y[i]",
               "0.05*n[i]", "em", 10, 0.02, 150, 30, 3),
    "funcs": (2, 3, 2, "exp(-abs(y[i]))*ln(2 + y[i]^2) + tan(0.1*y[i]) - p[0]*y[i] + 2^-3^2",
              "p[1 + i]*cos(y[i])*n[1 - i]", "em", 9, 0.01, 100, 25, 5),
    "rk4": (5, 6, 0, "p[0]*sum(j, (y[j] - y[i])*exp(-abs(y[j] - y[i]))) + p[1 + i] - 0.5*y[i]^2*t",
            "0", "rk4", 8, 0.02, 100, 10, 0),
    "euler": (3, 1, 0, "p[0] - ln(1 + y[i]*y[i]) + i", "0", "euler", 7, 0.05, 60, 15, 0),
    "fail": (2, 2, 2, "ln(y[i]) + p[0]", "p[1]*n[i]", "em", 6, 0.01, 80, 20, 9),
    "big": (40, 3, 40, "p[0]/N*sum(j, sin(y[j] - y[i])) + p[1]", "p[2]*n[i]", "em", 6, 0.01, 40,
            10, 2),
    "kuramoto": (8, 17, 8, model.KURAMOTO_DRIFT_TEMPLATE, model.KURAMOTO_DIFFUSION_TEMPLATE, "em",
                 10, 0.01, 100, 25, 4),
}

arrays: dict[str, np.ndarray] = {}
cases: dict[str, dict] = {}

for name, (n, npar, nn, drift, diff, solver, m, dt, steps, ks, seed) in MODELS.items():
    g = np.random.default_rng(zlib.crc32(name.encode()))
    init = g.uniform(-1.5, 1.5, size=(m, n))
    params = g.uniform(0.05, 0.6, size=(m, npar))
    if name == "fail":
        init[:, 0] = np.linspace(1.0, 0.2, m)
        init[m // 2:, 1] = -0.5   # ln of a negative phase -> NaN at step 0
        params[:, 0] = -30.0      # drives y[0] through 0 for the first half
    spec = model.model_from_dsl(name, n, npar, nn, drift, diff)
    cfg = EngineConfig(dt=dt, tspan=dt * steps, ksteps=ks, orbits=m, solver=solver, seed=seed)
    store = run_batch(spec, cfg, OrbitBatch(init=init, params=params))
    arrays[name + "_init"] = init
    arrays[name + "_params"] = params
    arrays[name + "_values"] = store.values
    cases[name] = dict(nequat=n, nparams=npar, nnoise=nn, drift=drift, diffusion=diff,
                       solver=solver, orbits=m, dt=dt, steps=steps, ksteps=ks, seed=seed,
                       failures=[[f.orbit, f.chunk, f.step, f.time, f.reason]
                                 for f in store.failures])
    # drift / diffusion evaluations at a random state and time
    y = g.standard_normal((5, n))
    p = g.uniform(0.05, 0.6, size=(5, npar))
    arrays[name + "_eval_y"] = y
    arrays[name + "_eval_p"] = p
    arrays[name + "_drift"] = model.drift_eval(spec, 0.37, y, p, strict=False)
    if nn:
        z = g.standard_normal((5, nn))
        arrays[name + "_eval_noise"] = z
        arrays[name + "_diffusion"] = model.diffusion_eval(spec, 0.37, y, p, z, strict=False)

np.savez_compressed(os.path.join(HERE, "golden_dsl_v1.npz"), **arrays)
with open(os.path.join(HERE, "cases_dsl.json"), "w") as f:
    json.dump(cases, f, indent=1, sort_keys=True)
print("wrote %d arrays, %d cases" % (len(arrays), len(cases)))
for k, c in cases.items():
    print(k, "failures:", len(c["failures"]))
