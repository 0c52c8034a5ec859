"""Small runs of every kernel variant, for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py CASE

Each case is a short run (a few thousand orbits, tens of steps) that still
exercises the code path the verdict asked about: the persistent slab
hand-off (ld.acquire / st.release spin-wait), the pairwise shared-memory
staging at one lane and at several lanes per orbit, the fused order
parameter, stateful streams, RK4, tiled host pipelines and the generated
(NVRTC) lane-group programs.  Every case checks its result against the
oracle, so a sanitizer-clean run is also a correct one.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1908_03869_b200 as sdb  # noqa: E402
from oracle import sdeb_oracle as O  # noqa: E402

TOL = 1e-10


def _check(store, batch, n, steps, ksteps, seed, stream="philox", solver="em", nnoise=None,
           rows=None):
    rows = list(range(min(8, batch.orbits))) + [batch.orbits - 1] if rows is None else rows
    _, want, _ = O.integrate(batch.init[rows], batch.params[rows], dt=1e-3, ksteps=ksteps,
                             chunks=steps // ksteps, seed=seed, solver=solver,
                             nnoise=n if nnoise is None else nnoise, stream=stream,
                             orbit_ids=np.asarray(rows, dtype=np.uint64))
    err = O.mixed_error(store.values[rows], want)
    assert err <= TOL, err
    return err


def _run(n, m, steps, ksteps, layout=None, seed=5, **cfg):
    if layout:
        os.environ["SDEB200_LAYOUT"] = layout
    else:
        os.environ.pop("SDEB200_LAYOUT", None)
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.4, seed=11)
    solver = cfg.pop("solver", "em")
    model = sdb.kuramoto_model(n)
    if solver == "rk4":
        model = sdb.ModelSpec(name="ode", nequat=n, nparams=2 * n + 1, nnoise=0,
                              drift=sdb.model._kuramoto_drift)
    c = sdb.EngineConfig(dt=1e-3, tspan=1e-3 * steps, ksteps=ksteps, orbits=m, seed=seed,
                         solver=solver, devices=(0,), **cfg)
    return batch, c, model


def case_persistent():
    # persistent work-pulling grid, 1 CTA/SM: 8 CTA-groups per SM, slabs of 16 steps
    batch, c, model = _run(16, 148 * 8 * 64, 64, 64, layout="2,1,1")
    store = sdb.run_batch(model, c, batch)
    _check(store, batch, 16, 64, 64, c.seed)


def case_grid():
    batch, c, model = _run(32, 4096, 40, 10, layout="2,0,0")
    _check(sdb.run_batch(model, c, batch), batch, 32, 40, 10, c.seed)


def case_padded():
    batch, c, model = _run(13, 2000, 30, 10, layout="4,0,0")
    _check(sdb.run_batch(model, c, batch), batch, 13, 30, 10, c.seed)


def case_exact():
    batch, c, model = _run(5, 3000, 30, 15, layout="1,0,0,0,5")
    _check(sdb.run_batch(model, c, batch), batch, 5, 30, 15, c.seed)


def case_pairwise_l1():
    batch, c, model = _run(16, 2048, 20, 10, layout="1,0,0", coupling="pairwise")
    _check(sdb.run_batch(model, c, batch), batch, 16, 20, 10, c.seed)


def case_pairwise_lanes():
    for lanes in (4, 8):
        batch, c, model = _run(32, 1024, 12, 6, coupling="pairwise", lanes=lanes)
        _check(sdb.run_batch(model, c, batch), batch, 32, 12, 6, c.seed)


def case_streams():
    for stream in ("sfc64", "xoshiro256pp"):
        batch, c, model = _run(8, 4096, 24, 8, layout="2,0,0", stream=stream)
        _check(sdb.run_batch(model, c, batch), batch, 8, 24, 8, c.seed, stream=stream)


def case_rk4():
    batch, c, model = _run(16, 2048, 12, 4, layout="4,0,0", solver="rk4")
    _check(sdb.run_batch(model, c, batch), batch, 16, 12, 4, c.seed, solver="rk4", nnoise=0)


def case_coherence():
    batch, c, model = _run(32, 2048, 30, 10, layout="2,0,0")
    fused = sdb.run_coherence(model, c, batch)
    post = sdb.coherence_series(sdb.run_batch(model, c, batch))
    assert np.array_equal(fused.r, post.r) and np.array_equal(fused.phi, post.phi)


def case_tiles():
    os.environ["SDEB200_TILES"] = "3"
    batch, c, model = _run(16, 9000, 20, 5, layout="2,0,0")
    c2 = sdb.EngineConfig(**{**c.__dict__, "devices": (0, 0)})
    store = sdb.run_batch(model, c2, batch)
    _check(store, batch, 16, 20, 5, c.seed)
    os.environ.pop("SDEB200_TILES")


def case_autotune():
    # the layout autotuner's probe launches (scratch buffers, every candidate)
    batch, c, model = _run(64, 4096, 32, 32)
    _check(sdb.run_batch(model, c, batch), batch, 64, 32, 32, c.seed)


def case_dsl():
    os.environ.pop("SDEB200_LAYOUT", None)
    os.environ["SDEB200_NO_NATIVE_KURAMOTO"] = "1"  # the generated program, not the stepper
    n, m = 24, 1024
    model = sdb.model_from_dsl("kt", n, 2 * n + 1, n, sdb.model.KURAMOTO_DRIFT_TEMPLATE,
                               sdb.model.KURAMOTO_DIFFUSION_TEMPLATE)
    batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.4, seed=3)
    for coupling in ("meanfield", "pairwise"):
        c = sdb.EngineConfig(dt=1e-3, tspan=0.02, ksteps=10, orbits=m, seed=2, coupling=coupling,
                             devices=(0,))
        store = sdb.run_batch(model, c, batch)
        _check(store, batch, n, 20, 10, 2)
    os.environ.pop("SDEB200_NO_NATIVE_KURAMOTO")


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or sorted(CASES)
    for name in names:
        CASES[name]()
        print("case %s ok" % name, flush=True)
