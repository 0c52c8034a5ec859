"""Batch execution on B200 (drop-in for ``sdebatch.engine``,
/root/reference/pkg/src/sdebatch/engine.py).

``run_batch`` keeps the reference's signature, validation order, error
messages, store layout and failure semantics; the chunk x step loop
(engine.py:223-263) runs as one fused CUDA kernel per device shard behind
the C ABI ``sdb_run`` (include/sdeb200.h).

Noise is addressed by the absolute step index exactly as in the reference
(engine.py:10-15), so results are bit-identical for any ``threads``,
``chunk_group``, device list or kernel lane layout, and a coarser ``ksteps``
gives exactly a subsample of a finer one.

New, optional fields on EngineConfig (defaults keep reference behaviour):
  stream   -- "philox" (the reference's generator, default), "sfc64" or
              "xoshiro256pp" (per-(orbit, block) streams).
  coupling -- "meanfield" (default; O(n) order-parameter form of the
              coupling sum) or "pairwise" (O(n^2), term-by-term as model.py:193).
  devices  -- GPU ids to shard orbits over (default: SDEB200_DEVICES or (0,)).
  lanes    -- threads per orbit (power of two) or 0 to autotune.
"""

from __future__ import annotations

import ctypes
import dataclasses
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .model import (ModelSpec, OrbitBatch, expression_model, kuramoto_signature,
                    require_device_model)
from .solvers import get_solver

__all__ = [
    "ConfigError", "EngineConfig", "TrajectoryStore", "OrbitFailure",
    "iteration_count", "partition_orbits", "run_batch", "shard_bounds", "run_batch_sharded",
]

_MASK32 = 0xFFFFFFFF
_MASK64 = 0xFFFFFFFFFFFFFFFF


class ConfigError(ValueError):
    """A run configuration that cannot be executed as requested (engine.py:40-41)."""


@dataclass(frozen=True)
class EngineConfig:
    """Description of one integration run (engine.py:44-85)."""

    dt: float
    tspan: float
    ksteps: int
    orbits: int
    solver: str = "em"
    chunk_group: int = 8
    seed: int = 0
    threads: int | str = "all"
    pad: bool = False
    solver_tol: float = 1e-10
    solver_max_iter: int = 50
    max_store_bytes: int = 4 * 2 ** 30
    stream: str = "philox"
    coupling: str = "meanfield"
    devices: tuple | None = None
    lanes: int = 0

    def __post_init__(self):
        if self.dt <= 0:
            raise ConfigError("dt must be positive")
        if self.tspan <= 0:
            raise ConfigError("tspan must be positive")
        if self.ksteps < 1:
            raise ConfigError("ksteps must be >= 1")
        if self.orbits < 1:
            raise ConfigError("orbits must be >= 1")
        if self.chunk_group < 1:
            raise ConfigError("chunk_group must be >= 1")
        get_solver(self.solver)
        if self.threads != "all":
            if not isinstance(self.threads, int) or self.threads < 1:
                raise ConfigError("threads must be a positive integer or 'all'")
        if self.stream not in nat.STREAM_IDS:
            raise ConfigError("unknown noise stream %r (choose from %s)"
                              % (self.stream, ", ".join(sorted(nat.STREAM_IDS))))
        if self.coupling not in nat.COUPLING_IDS:
            raise ConfigError("unknown coupling evaluation %r (choose from %s)"
                              % (self.coupling, ", ".join(sorted(nat.COUPLING_IDS))))
        if self.lanes not in (0, 1, 2, 4, 8, 16, 32):
            raise ConfigError("lanes must be 0 (autotune) or a power of two <= 32")
        if self.devices is not None:
            devs = tuple(self.devices)
            if not devs or any((not isinstance(d, int)) or d < 0 for d in devs):
                raise ConfigError("devices must be a non-empty tuple of GPU ids")
            object.__setattr__(self, "devices", devs)

    def worker_count(self) -> int:
        """engine.py:82-85 (a scheduling hint only; never changes results)."""
        if self.threads == "all":
            return os.cpu_count() or 1
        return self.threads


@dataclass(frozen=True)
class OrbitFailure:
    """First solver failure of one orbit; the rest of its row is NaN (engine.py:88-96)."""

    orbit: int
    chunk: int
    step: int
    time: float
    reason: str


@dataclass
class TrajectoryStore:
    """Sampled states of every orbit (engine.py:99-123): ``values`` is
    (orbits, samples, nequat), sample 0 the initial state verbatim."""

    times: np.ndarray
    values: np.ndarray
    model_name: str = ""
    config: EngineConfig | None = None
    failures: list = field(default_factory=list)

    @property
    def orbits(self) -> int:
        return self.values.shape[0]

    @property
    def samples(self) -> int:
        return self.values.shape[1]

    @property
    def nequat(self) -> int:
        return self.values.shape[2]


def iteration_count(tspan: float, dt: float, ksteps: int, pad: bool = False) -> int:
    """Number of chunks k = tspan / (dt * ksteps) (engine.py:126-142)."""
    if dt <= 0 or tspan <= 0 or ksteps < 1:
        raise ConfigError("tspan, dt and ksteps must be positive")
    ratio = tspan / (dt * ksteps)
    k = round(ratio)
    if k >= 1 and abs(ratio - k) <= 1e-9 * max(1.0, abs(ratio)):
        return k
    if pad:
        return max(1, math.ceil(ratio - 1e-12))
    raise ConfigError(
        "tspan=%g is not an integer multiple of dt*ksteps=%g (pass pad=True to round up)"
        % (tspan, dt * ksteps))


def partition_orbits(orbits: int, chunk_group: int) -> list[range]:
    """Contiguous orbit ranges of width chunk_group (engine.py:145-150)."""
    if orbits < 1 or chunk_group < 1:
        raise ConfigError("orbits and chunk_group must be >= 1")
    return [range(start, min(start + chunk_group, orbits))
            for start in range(0, orbits, chunk_group)]


def _check_stepper(model: ModelSpec, config: EngineConfig):
    """engine.py:153-160: a deterministic solver on a noisy model is an error."""
    info = get_solver(config.solver)
    if not info.stochastic and model.nnoise > 0:
        raise ConfigError(
            "solver %r is deterministic but model %r has %d noise terms; "
            "use the em solver or a noise-free model"
            % (config.solver, model.name, model.nnoise))
    if info.implicit:
        raise NotImplementedError(
            "implicit solver %r is outside the device path (em/euler/rk4 only)" % (config.solver,))
    return info


def make_desc(model: ModelSpec, config: EngineConfig, chunks: int, orbits: int,
              orbit_offset: int = 0) -> nat.SdbDesc:
    """Descriptor for the C ABI (include/sdeb200.h sdb_desc)."""
    require_device_model(model)
    sig = kuramoto_signature(model)
    n, nnoise = sig if sig is not None else (model.nequat, model.nnoise)
    d = nat.SdbDesc()
    d.model = nat.SDB_MODEL_KURAMOTO if sig is not None else nat.SDB_MODEL_EXPRESSION
    d.nequat = n
    d.nparams = model.nparams
    d.nnoise = nnoise
    d.solver = nat.SOLVER_IDS[config.solver]
    d.stream = nat.STREAM_IDS[config.stream]
    d.coupling = nat.COUPLING_IDS[config.coupling]
    d.lanes = int(config.lanes)
    d.seed = int(config.seed) & _MASK64
    d.dt = float(config.dt)
    d.ksteps = int(config.ksteps)
    d.chunks = int(chunks)
    d.orbits = int(orbits)
    d.orbit_offset = int(orbit_offset)
    return d


def failures_from_steps(fail_step: np.ndarray, ksteps: int, dt: float,
                        orbit_offset: int = 0) -> list[OrbitFailure]:
    """Per-orbit first-failure steps -> OrbitFailure records sorted by orbit
    (engine.py:257-261, 275)."""
    out = []
    for idx in np.nonzero(fail_step >= 0)[0]:
        s = int(fail_step[idx])
        out.append(OrbitFailure(orbit=orbit_offset + int(idx), chunk=s // ksteps,
                                step=s % ksteps, time=s * dt,
                                reason="state became non-finite"))
    return out


def shard_bounds(orbits: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [r*M/W, (r+1)*M/W) of rank r -- the same split sdb_run
    uses across the devices of one context."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError("bad shard rank %r of world %r" % (rank, world))
    return rank * orbits // world, (rank + 1) * orbits // world


def validate_run(model: ModelSpec, config: EngineConfig, batch: OrbitBatch, orbit_offset: int = 0,
                 store_cap: bool = True) -> int:
    """run_batch's checks in the reference's order (engine.py:192-210); returns
    the chunk count.  ``store_cap=False`` skips the trajectory-store size cap
    (runs that never materialise the store, e.g. analysis.run_coherence)."""
    batch.check_against(model)
    if batch.orbits != config.orbits:
        raise ConfigError("config says %d orbits but batch has %d"
                          % (config.orbits, batch.orbits))
    if batch.orbits > _MASK32:
        raise ConfigError("orbit count must fit in 32 bits")
    if orbit_offset < 0 or orbit_offset + batch.orbits > _MASK32 + 1:
        raise ConfigError("global orbit ids must fit in 32 bits")
    chunks = iteration_count(config.tspan, config.dt, config.ksteps, pad=config.pad)
    if chunks * config.ksteps >= 2 ** 63:
        raise ConfigError("total step count does not fit in 63 bits")

    samples = chunks + 1
    store_bytes = batch.orbits * samples * model.nequat * 8
    if store_cap and store_bytes > config.max_store_bytes:
        raise ConfigError(
            "trajectory store would need %d bytes (orbits=%d, samples=%d, nequat=%d), "
            "above the configured cap of %d"
            % (store_bytes, batch.orbits, samples, model.nequat, config.max_store_bytes))
    _check_stepper(model, config)
    return chunks


def run_batch(model: ModelSpec, config: EngineConfig, batch: OrbitBatch, *,
              orbit_offset: int = 0) -> TrajectoryStore:
    """Integrate every orbit of the batch on the GPU and sample once per chunk
    (engine.py:184-277).  Validation happens before any device allocation,
    in the reference's order.

    ``orbit_offset`` (keyword, default 0 = the reference's numbering) is the
    global id of row 0: noise is keyed by global id and failures report it, so
    a shard of a larger batch integrates exactly as those rows of the whole.
    """
    chunks = validate_run(model, config, batch, orbit_offset)
    samples = chunks + 1
    desc = make_desc(model, config, chunks, batch.orbits, orbit_offset)
    if desc.model == nat.SDB_MODEL_EXPRESSION:
        # indices are checked up front: the reference raises DomainError at step 0
        from . import program
        program.check_model_indices(model)

    sample_dt = config.ksteps * config.dt
    times = np.arange(samples, dtype=np.float64) * sample_dt
    values = nat.host_empty((batch.orbits, samples, model.nequat))
    fail_step = np.empty(batch.orbits, dtype=np.int64)
    init = nat.f64(batch.init)
    params = nat.f64(batch.params)
    ctx = nat.context(config.devices)
    if desc.model == nat.SDB_MODEL_EXPRESSION:
        cm = program.model_program(model)  # compiled expression-template program
        nat.check(nat.lib().sdb_run_model(ctx, cm.handle, desc, nat.dptr(init), nat.dptr(params),
                                          nat.dptr(values), nat.i64ptr(fail_step)),
                  ctx, "sdb_run_model")
    else:
        nat.check(nat.lib().sdb_run(ctx, desc, nat.dptr(init), nat.dptr(params),
                                    nat.dptr(values), nat.i64ptr(fail_step)), ctx, "sdb_run")
    failures = failures_from_steps(fail_step, config.ksteps, config.dt, orbit_offset)
    return TrajectoryStore(times=times, values=values, model_name=model.name,
                           config=config, failures=failures)


def run_batch_sharded(model: ModelSpec, config: EngineConfig, batch: OrbitBatch, *,
                      world: int, rank: int, devices=None, gather=None) -> TrajectoryStore:
    """Multi-process form (one process per GPU, e.g. under torchrun): rank r
    integrates rows shard_bounds(M, world, r) of ``batch`` on its device(s)
    with their global orbit ids.  There is no collective on the data path;
    ``gather`` (e.g. a torch.distributed all_gather_object wrapper) may
    assemble the full store on the host afterwards.  The assembled store is
    bit-identical to a single-process run (noise is keyed by global id)."""
    # every rank validates the whole run first: a bad configuration raises on
    # all ranks alike, before any of them reaches the collective in ``gather``
    chunks = validate_run(model, config, batch)
    lo, hi = shard_bounds(batch.orbits, world, rank)
    if hi > lo:
        part = OrbitBatch(init=batch.init[lo:hi], params=batch.params[lo:hi])
        cfg = dataclasses.replace(config, orbits=hi - lo,
                                  devices=devices if devices is not None else config.devices)
        store = run_batch(model, cfg, part, orbit_offset=lo)
    else:  # more ranks than orbits: this rank's shard is empty, it still joins the gather
        times = np.arange(chunks + 1, dtype=np.float64) * (config.ksteps * config.dt)
        store = TrajectoryStore(times=times, values=np.empty((0, chunks + 1, model.nequat)),
                                model_name=model.name, config=config, failures=[])
    if gather is None:
        return store
    parts = gather((lo, store.values, store.failures))
    parts.sort(key=lambda t: t[0])
    values = np.concatenate([p[1] for p in parts], axis=0)
    failures = sorted((f for p in parts for f in p[2]), key=lambda f: f.orbit)
    return TrajectoryStore(times=store.times, values=values, model_name=model.name,
                           config=config, failures=failures)


def last_launch_info(devices=None) -> dict:
    """Kernel launches and lane layout of the most recent run on a context."""
    ctx = nat.context(devices)
    lib = nat.lib()
    lay = [ctypes.c_int32() for _ in range(5)]
    lib.sdb_last_layout(ctx, *(ctypes.byref(v) for v in lay))
    lanes, persistent, ctas, variant, tiles = (int(v.value) for v in lay)
    return {"launches": int(lib.sdb_last_launch_count(ctx)), "lanes": lanes,
            "tune_us": int(lib.sdb_last_tune_us(ctx)),
            "lane_width": int(lib.sdb_last_lane_width(ctx)),
            "persistent_grid": bool(persistent), "ctas_per_sm": ctas,
            "register_capped": bool(variant), "tiles": tiles}
