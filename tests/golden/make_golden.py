"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``sdebatch`` from /root/reference/pkg/src and records, for small
seeded inputs, the reference's own outputs on the hot path:
Philox words, per-step normals, sampling uniforms / sampled batches, drift
evaluations and complete ``run_batch`` trajectory stores (em / euler / rk4,
failures, pad, wrapped seeds).  The output ``golden_v1.npz`` + ``cases.json``
are committed; tests read them on any machine (the GPU box has no
/root/reference).
"""

from __future__ import annotations

import dataclasses
import json
import math
import os
import sys

import numpy as np

REF = os.environ.get("SDEBATCH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from sdebatch import model, rng  # noqa: E402
from sdebatch.engine import EngineConfig, run_batch  # noqa: E402
from sdebatch.model import ModelSpec, OrbitBatch  # noqa: E402
from sdebatch.storage import store_hash  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ACCEPT_SEED = 20260809

arrays: dict[str, np.ndarray] = {}
cases: dict[str, dict] = {}


def put(name, arr):
    arrays[name] = np.ascontiguousarray(arr)


# -- Philox words over random keys/counters --------------------------------
g = np.random.default_rng(1234)
kc = g.integers(0, 2 ** 32, size=(256, 6), dtype=np.uint64).astype(np.uint32)
words = rng._philox_words(kc[:, 0], kc[:, 1], kc[:, 2], kc[:, 3], kc[:, 4], kc[:, 5])
put("philox_in", kc)
put("philox_out", np.stack(words, axis=-1))

# -- per-step normals at assorted addresses --------------------------------
normal_cases = [(0, 0, 0, 4), (42, 0, 5, 7), (2 ** 63, 0, 1, 1), (5, 4, 2, 12),
                (ACCEPT_SEED, 0, 9999, 16), (2 ** 64 - 1, 1, 3, 33), (123, 0, 7, 256)]
for idx, (seed, chunk, step, m) in enumerate(normal_cases):
    orbits = np.array([0, 1, 2, 17, 1023, 65535, 2 ** 32 - 1], dtype=np.uint32)
    put("normals_%d" % idx, rng.normals_for_orbits(seed, orbits, chunk, step, m))
    cases["normals_%d" % idx] = dict(seed=str(seed), chunk=chunk, step=step, m=m,
                                     orbits=[int(o) for o in orbits])

# -- sampling uniforms and sampled batches ---------------------------------
put("sampling_uniforms", rng.sampling_uniforms(11, np.arange(8, dtype=np.uint32), 10))
b = model.sample_kuramoto_batch(16, 64, (0.2, 0.4), (0.01, 0.03), 0.25, seed=99)
put("sample_init", b.init)
put("sample_params", b.params)
b = model.speed_protocol_batch(4, 32, seed=ACCEPT_SEED)
put("speed_init", b.init)
put("speed_params", b.params)

# -- drift evaluations ------------------------------------------------------
for n in (1, 2, 3, 8, 16, 33, 64):
    y = g.uniform(-4 * math.pi, 4 * math.pi, (6, n))
    p = np.column_stack([g.uniform(0, 1, 6), g.uniform(0.2, 0.4, (6, n)),
                         g.uniform(0.01, 0.03, (6, n))])
    km = model.kuramoto_model(n)
    put("drift_y_%d" % n, y)
    put("drift_p_%d" % n, p)
    put("drift_f_%d" % n, model.drift_eval(km, 0.0, y, p))


# -- full run_batch stores ---------------------------------------------------
def store_case(name, m, batch, config, note):
    store = run_batch(m, config, batch)
    put(name + "_init", batch.init)
    put(name + "_params", batch.params)
    put(name + "_times", store.times)
    put(name + "_values", store.values)
    cfg = dataclasses.asdict(config)
    cfg["seed"] = str(config.seed)
    cases[name] = dict(config=cfg, nequat=m.nequat, nparams=m.nparams, nnoise=m.nnoise,
                       model=m.name, note=note, sha256=store_hash(store),
                       failures=[[f.orbit, f.chunk, f.step, f.time, f.reason]
                                 for f in store.failures])


def kgrid_batch(n, orbits, seed, ks, sigmas, omega=(0.2, 0.4)):
    b = model.sample_kuramoto_batch(n, orbits, omega, (0.01, 0.03), 0.0, seed=seed)
    params = b.params.copy()
    params[:, 0] = ks[np.arange(orbits) // len(sigmas) % len(ks)]
    params[:, n + 1:] = sigmas[np.arange(orbits) % len(sigmas)][:, None]
    return OrbitBatch(init=b.init, params=params)


km4 = model.kuramoto_model(4)
store_case("cfg1", km4, model.speed_protocol_batch(4, 64, seed=ACCEPT_SEED),
           EngineConfig(dt=1e-3, tspan=1.0, ksteps=100, orbits=64, seed=ACCEPT_SEED),
           "config 1 shape, 1000 steps, sample every 100")

km5 = model.kuramoto_model(5)
b5 = model.sample_kuramoto_batch(5, 16, (0.2, 0.4), (0.01, 0.03), 0.2, seed=7)
store_case("engine5", km5, b5,
           EngineConfig(dt=0.05, tspan=4.0, ksteps=8, orbits=16, seed=3),
           "test_engine.py kuramoto_setup, ksteps=8")
store_case("engine5_k4", km5, b5,
           EngineConfig(dt=0.05, tspan=4.0, ksteps=4, orbits=16, seed=3),
           "ksteps subsampling identity partner")

km16 = model.kuramoto_model(16)
b16 = kgrid_batch(16, 64, 5, np.linspace(0.0, 0.5, 8), np.geomspace(1e-3, 1e-1, 8))
store_case("cfg2", km16, b16,
           EngineConfig(dt=1e-3, tspan=2.0, ksteps=500, orbits=64, seed=ACCEPT_SEED),
           "config 2 shape (K x sigma grid), 2000 steps")

km33 = model.kuramoto_model(33)
store_case("n33", km33, model.sample_kuramoto_batch(33, 8, (0.2, 0.4), (0.01, 0.03), 0.4, seed=3),
           EngineConfig(dt=0.01, tspan=2.0, ksteps=50, orbits=8, seed=2 ** 64 - 1),
           "ragged n=33 (not a multiple of 4), seed 2**64-1")

km64 = model.kuramoto_model(64)
store_case("n64", km64, model.speed_protocol_batch(64, 4, seed=1),
           EngineConfig(dt=1e-3, tspan=0.2, ksteps=100, orbits=4, seed=-5),
           "n=64, negative seed wraps mod 2**64")

km256 = model.kuramoto_model(256)
store_case("n256", km256, model.speed_protocol_batch(256, 2, seed=2),
           EngineConfig(dt=1e-3, tspan=0.02, ksteps=10, orbits=2, seed=17),
           "n=256 config 3 shape, 20 steps")

ode8 = ModelSpec(name="kuramoto-ode:8", nequat=8, nparams=17, nnoise=0,
                 drift=model._kuramoto_drift)
b8 = kgrid_batch(8, 16, 11, np.linspace(0.0, 2.0, 4), np.zeros(4))
store_case("rk4_8", ode8, b8,
           EngineConfig(dt=1e-2, tspan=2.0, ksteps=20, orbits=16, solver="rk4"),
           "deterministic Kuramoto (nnoise=0) with rk4")
store_case("euler_8", ode8, b8,
           EngineConfig(dt=1e-2, tspan=2.0, ksteps=20, orbits=16, solver="euler"),
           "deterministic Kuramoto (nnoise=0) with euler")
store_case("em0_8", ode8, b8,
           EngineConfig(dt=1e-2, tspan=2.0, ksteps=20, orbits=16, solver="em"),
           "em on a nnoise=0 model == euler")

km2 = model.kuramoto_model(2)
fail_init = np.array([[np.inf, 0.0], [0.1, 0.2], [0.0, 0.0], [0.3, -0.3]])
fail_params = np.array([[0.5, 0.1, 0.2, 0.01, 0.01],
                        [0.5, 0.1, 0.2, 0.01, 0.01],
                        [0.0, 1e308, 0.2, 0.0, 0.0],
                        [0.5, 0.1, 0.2, 0.01, 0.01]])
store_case("failures", km2, OrbitBatch(init=fail_init, params=fail_params),
           EngineConfig(dt=0.5, tspan=4.0, ksteps=2, orbits=4, seed=1),
           "orbit 0 fails at step 0 (inf init); orbit 2 overflows at step 3")

km1 = model.kuramoto_model(1)
store_case("pad", km1, OrbitBatch(init=np.array([[0.0]]), params=np.array([[0.0, 0.3, 0.0]])),
           EngineConfig(dt=0.3, tspan=1.0, ksteps=1, orbits=1, pad=True),
           "pad rounds the chunk count up")
store_case("rotator", km1, OrbitBatch(init=np.array([[0.5]]), params=np.array([[0.0, 0.3, 0.0]])),
           EngineConfig(dt=0.05, tspan=10.0, ksteps=20, orbits=1, seed=1),
           "single uncoupled rotator")

km10 = model.kuramoto_model(10)
store_case("accept7", km10, model.accuracy_protocol_batch(10, 64, 0.2, seed=ACCEPT_SEED),
           EngineConfig(dt=0.05, tspan=40.0, ksteps=40, orbits=64, seed=ACCEPT_SEED),
           "acceptance criterion 7 shape (64 of the 512 orbits), 800 steps")

np.savez_compressed(os.path.join(HERE, "golden_v1.npz"), **arrays)
with open(os.path.join(HERE, "cases.json"), "w") as fh:
    json.dump(cases, fh, indent=1, sort_keys=True)
print("wrote %d arrays, %d cases" % (len(arrays), len(cases)))
