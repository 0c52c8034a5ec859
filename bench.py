#!/usr/bin/env python
"""Benchmark: orbit-steps/s of stochastic Kuramoto Euler-Maruyama on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg3] [--coupling meanfield|pairwise]

BASELINE.json's metric is "orbit-steps/s ... 1/2/4/8 B200"; the config it
names at 1/2/4/8 GPUs is configs[2] (cfg3): stochastic Kuramoto n = 32, 64,
128, 256, 2^20 orbits each, Philox, dt = 1e-3, final state.  The default
workload "cfg3" runs all four sizes; the headline line is the largest
(n = 256, 100 steps), the other sizes are under "sizes", and cfg2
(BASELINE configs[1], n = 16, 65,536 orbits, sfc64, 10^4 steps) is under
"secondary".

One "step" = one complete run of the workload (all orbits x all SDE steps).
Scaling is STRONG: the fixed batch of the workload is split into contiguous
orbit shards [g*M/N, (g+1)*M/N) with their global orbit ids,
so the results are bit-identical for any N.  N GPUs:
  * under torchrun (WORLD_SIZE = N): one process per GPU, rank r runs shard
    r on LOCAL_RANK; time = max over ranks (NCCL all-reduce of one float,
    timing only -- the data path has no collective);
  * without torchrun, --gpus N > 1: one process drives N devices, the
    device-resident leg launches every shard on its own device's stream, the
    e2e leg is run_batch with EngineConfig(devices=range(N)) (the drop-in
    path: one host thread per device inside libsdeb200).

  value     device-resident inputs (sdb_run_device), CUDA events on the launch
            stream around each launch, L2 flushed (512 MiB memset) between
            timed steps outside the event pairs; max over GPUs per step.
  e2e       the public API run_batch() with numpy host buffers: H2D of
            init/params and D2H of the store inside every timed step.
  cold_e2e  the first run_batch() call of a fresh process (its own subprocess,
            empty layout cache): everything a one-shot CLI call pays.
  roofline  FP64 pipe: "frac" = the kernel's own algorithmic FP64 lane-ops
            (the O(n) meanfield form) / kernel time, against the
            FP64 DFMA peak measured live (sdb_fp64_peak; MEASURED_PEAKS.json
            has no FP64 figure); "w_em_frac" = the same time against SURVEY.md
            8d's W_EM(n) = 9n(n-1) + 41n of the reference's O(n^2) algorithm.
  cpu_baseline  the UNMODIFIED reference (sdebatch.run_batch from
            baseline/_ref, its own bench.time_run protocol) on a bounded
            sample, threads = 1 and threads = "all", best chunk_group of
            {M_cpu, M_cpu/threads, 8192, 512} each; the oracle
            port only if baseline/_ref is absent ("kind" says which).
--impl reference times that reference alone (rank 0, all host threads).
"""

from __future__ import annotations

import argparse
import gc
import hashlib
import json
import os
import platform
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
REF_PATH = os.path.join(ROOT, "baseline", "_ref")

WORKLOADS = {
    # BASELINE.json configs[2] -- the headline (the config stated at 1/2/4/8 GPUs)
    "cfg3": dict(sizes=("cfg3_n32", "cfg3_n64", "cfg3_n128", "cfg3_n256"),
                 headline="cfg3_n256", secondary=("cfg2",),
                 desc="stochastic Kuramoto size sweep n=32..256, 2^20 orbits, Philox, "
                      "E-M dt=1e-3, final state (headline: n=256)"),
    # BASELINE.json configs[1]
    "cfg2": dict(n=16, orbits=65536, dt=1e-3, steps=10000, ksteps=10000, stream="sfc64",
                 solver="em", batch="kgrid",
                 desc="stochastic Kuramoto n=16, 65,536 orbits (256 K x 256 sigma grid), sfc64, "
                      "E-M dt=1e-3, 10^4 steps, final state only"),
    "cfg1": dict(n=4, orbits=1024, dt=1e-3, steps=10000, ksteps=10000, stream="xoshiro256pp",
                 solver="em", batch="speed", desc="n=4, 1,024 orbits, xoshiro256++, 10^4 steps"),
    "cfg3_n32": dict(n=32, orbits=1 << 20, dt=1e-3, steps=1000, ksteps=1000, stream="philox",
                     solver="em", batch="speed", desc="n=32, 2^20 orbits, 1000 steps"),
    "cfg3_n64": dict(n=64, orbits=1 << 20, dt=1e-3, steps=1000, ksteps=1000, stream="philox",
                     solver="em", batch="speed", desc="n=64, 2^20 orbits, 1000 steps"),
    "cfg3_n128": dict(n=128, orbits=1 << 20, dt=1e-3, steps=200, ksteps=200, stream="philox",
                      solver="em", batch="speed", desc="n=128, 2^20 orbits, 200 steps"),
    "cfg3_n256": dict(n=256, orbits=1 << 20, dt=1e-3, steps=100, ksteps=100, stream="philox",
                      solver="em", batch="speed", desc="n=256, 2^20 orbits, 100 steps"),
    "cfg4": dict(n=64, orbits=1 << 18, dt=1e-3, steps=1000, ksteps=1000, stream="philox",
                 solver="rk4", batch="kgrid_ode",
                 desc="deterministic Kuramoto n=64, RK4, 2^18 orbits (512 K x 512 omega draws)"),
    "cfg5": dict(n=32, orbits=131072, dt=1e-3, steps=1000, ksteps=10, stream="philox",
                 solver="em", batch="resample",
                 desc="n=32, 512 parameter sets x 256 realisations, trajectory every 10 steps"),
    # the paper's own speed protocol: K = 1, omega ~ U[0.01, 0.03],
    # p ~ U[0.001, 0.003], dt = 0.05, 400 s = 8000 steps, FP64, largest M = 163,840 orbits;
    # BASELINE.md section 2 lists SODECL's published times (P100, 2x Xeon Gold 6142, ...)
    "paper_n5": dict(n=5, orbits=163840, dt=0.05, steps=8000, ksteps=8000, stream="philox",
                     solver="em", batch="speed", published=163840 * 8000 / 4.719,
                     desc="paper protocol N=5, M=163,840, dt=0.05, 8000 steps (P100: 4.719 s)"),
    "paper_n10": dict(n=10, orbits=163840, dt=0.05, steps=8000, ksteps=8000, stream="philox",
                      solver="em", batch="speed", published=163840 * 8000 / 9.315,
                      desc="paper protocol N=10, M=163,840, dt=0.05, 8000 steps (P100: 9.315 s)"),
    "paper_n15": dict(n=15, orbits=163840, dt=0.05, steps=8000, ksteps=8000, stream="philox",
                      solver="em", batch="speed", published=163840 * 8000 / 17.656,
                      desc="paper protocol N=15, M=163,840, dt=0.05, 8000 steps (P100: 17.656 s)"),
    # run_batch fused with coherence_series: only (r, Phi) per sample leaves
    # the GPU; the e2e line includes the D2H of that instead of the 3.2 GiB store
    "cfg5_coherence": dict(n=32, orbits=131072, dt=1e-3, steps=1000, ksteps=10, stream="philox",
                           solver="em", batch="resample", coherence=True,
                           desc="cfg5 through analysis.run_coherence: order parameter of every "
                                "10th step fused into the stepper"),
    # expression-template models through the NVRTC-generated program
    "cfg2_codegen": dict(n=16, orbits=65536, dt=1e-3, steps=10000, ksteps=10000, stream="sfc64",
                         solver="em", batch="kgrid", model="kuramoto_template",
                         desc="cfg2 through the generated program of the Kuramoto templates "
                              "(model_from_dsl, n^2 sin terms in the reference's order)"),
    "ou_codegen": dict(n=16, orbits=65536, dt=1e-3, steps=10000, ksteps=1000, stream="philox",
                       solver="em", batch="uniform", model="ou",
                       desc="Ornstein-Uhlenbeck template model (drift p[0]*(p[1]-y[i]), "
                            "diffusion p[2+i]*n[i]), n=16, 65,536 orbits, 10 samples"),
}
DEFAULT_WORKLOAD = "cfg3"

# expression-template workloads: (drift, diffusion, nparams(n))
TEMPLATES = {
    "kuramoto_template": ("p[i+1] + (p[0]/N) * sum(j, sin(y[j] - y[i]))", "p[1+N+i] * n[i]",
                          lambda n: 2 * n + 1),
    "ou": ("p[0]*(p[1] - y[i])", "p[2 + i]*n[i]", lambda n: n + 2),
}


SINCOS_OPS = 14      # csrc/sdeb_math.cuh sincos_tab: 4 reduction + 6 poly + 4 rotation
SIN_OPS = 12         # the same when only sin is used (the cos rotation is dead code)
BOX_MULLER_PAIR = 34  # uniform 1, -2*log 11 (the -2 folded into the table), sqrt 8, angle from the word 2, sincos poly+rotation 10, 2 products


def template_fp64_ops(n: int, model: str, coupling: str = "meanfield") -> float:
    """FP64 lane-ops per orbit-step of the generated program (counted from the
    generated code).  Kuramoto templates, literal form (coupling="pairwise"):
    n^2 terms x (difference 1, sin SIN_OPS, sum 1); factored form (meanfield):
    one sincos (SINCOS_OPS) + 2 sum adds per oscillator in the prologue (its
    (sin, cos) kept for the equations), then per equation the addition formula
    3.  Both: per equation p[0]/N, *, + 3, diffusion product 1, noise
    BOX_MULLER_PAIR / 2, update 4.  OU per equation drift 2 + diffusion 1 +
    noise + update 4."""
    tail = 1 + BOX_MULLER_PAIR / 2 + 4
    if model == "kuramoto_template":
        if coupling == "meanfield":
            return n * (SINCOS_OPS + 2) + n * (3 + 3 + tail)
        return n * n * (1 + SIN_OPS + 1) + n * (3 + tail)
    return n * (2 + tail)


def algorithmic_fp64_ops(n: int, solver: str, coupling: str) -> float:
    """FP64 lane-ops (DFMA/DMUL/DADD) per orbit-step of the algorithm the
    kernel runs, counted from the device code.
    Meanfield: sincos 14 + tree sums 2 per oscillator.  em (folded): the two
    scaled sums 2 per orbit, increment fma(cos, K/n dt sum sin, fma(-sin, .,
    omega dt)) 2 and update fma(sqrt(dt) s, N, y + inc) 2 per oscillator, plus
    Box-Muller 34 per pair of normals; rk4: 4 folded drifts (2 + 2/osc on the
    sums) + 13/osc; euler: the exact drift (S_i 3, omega + K/n S 2) + update 2.
    Pairwise: 15 per unordered pair (difference, sin 12, 2 accumulates) + 2/osc
    and the unfolded em update 5."""
    if coupling == "meanfield":
        sums = n * (SINCOS_OPS + 2)
        if solver == "em":
            return sums + 2 + n * (2 + 2 + BOX_MULLER_PAIR / 2)
        if solver == "rk4":
            return 4 * (sums + 2 + 2 * n) + n * 13
        return sums + n * (3 + 2) + n * 2
    drift = n * (n - 1) / 2 * (1 + SIN_OPS + 2) + n * 2
    if solver == "em":
        return drift + n * (5 + BOX_MULLER_PAIR / 2)
    if solver == "rk4":
        return 4 * drift + n * 13
    return drift + n * 2


def measured_traffic(workload: str):
    """DRAM bytes per launch from the committed ncu capture (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(workload, {}).get("dram_bytes")
    except (OSError, ValueError):
        return None


def pairwise_equivalent_ops(n: int) -> float:
    """SURVEY.md 8d W_EM(n) = 9 n(n-1) + 41 n (the reference algorithm's work)."""
    return 9.0 * n * (n - 1) + 41.0 * n


# ---------------------------------------------------------------------------
# workload construction (shards: rows [lo, hi) of the workload, global ids)

SEED = 20260809


def _shape_batch(make, w, lo, hi, sample):
    """The workload's batch rows [lo, hi).  ``sample(count, omega, noise, K,
    first)`` draws rows [first, first + count) of the counter-based Kuramoto
    sampler (model.py:242-270; bit-exact on the device), ``make(init,
    params)`` builds the OrbitBatch."""
    n = w["n"]
    rows = np.arange(lo, hi)
    m = hi - lo
    if w["batch"] == "speed":  # speed_protocol_batch (model.py:273-277)
        b = sample(m, (0.01, 0.03), (0.001, 0.003), 1.0, lo)
        return make(b.init, b.params)
    if w["batch"] == "kgrid":  # 256 K x 256 sigma
        b = sample(m, (0.2, 0.4), (0.01, 0.03), 0.0, lo)
        params = b.params.copy()
        params[:, 0] = np.linspace(0.0, 0.5, 256)[(rows // 256) % 256]
        params[:, n + 1:] = np.geomspace(1e-3, 1e-1, 256)[rows % 256][:, None]
        return make(b.init, params)
    if w["batch"] == "kgrid_ode":  # cfg4: 512 K x 512 omega draws, zero diffusion
        b = sample(m, (0.2, 0.4), (0.0, 0.0), 0.0, lo)
        params = b.params.copy()
        params[:, 0] = np.linspace(0.0, 2.0, 512)[(rows // 512) % 512]
        return make(b.init, params)
    if w["batch"] == "resample":  # cfg5: 512 parameter sets x 256 realisations
        s0, s1 = lo // 256, (hi - 1) // 256 + 1
        b = sample(s1 - s0, (0.2, 0.4), (0.01, 0.03), 0.0, s0)
        params = b.params.copy()
        params[:, 0] = np.linspace(0.05, 0.8, 16)[np.arange(s0, s1) % 16]
        cut = slice(lo - s0 * 256, hi - s0 * 256)
        return make(np.repeat(b.init, 256, axis=0)[cut], np.repeat(params, 256, axis=0)[cut])
    if w["batch"] == "uniform":  # generic template models: seeded uniform draws
        g = np.random.default_rng(SEED)
        nparams = TEMPLATES[w["model"]][2](n)
        init = g.uniform(-1.0, 1.0, (w["orbits"], n))
        params = g.uniform(0.05, 0.5, (w["orbits"], nparams))
        return make(init[lo:hi], params[lo:hi])
    raise ValueError(w["batch"])


def make_batch(sdb, w, lo: int = 0, hi: int | None = None):
    """Rows [lo, hi) of workload w's batch (default: all), drawn on the GPU."""
    hi = w["orbits"] if hi is None else hi

    def sample(count, omega, noise, k, first):
        return sdb.sample_kuramoto_batch(w["n"], count, omega, noise, k, SEED, orbit_offset=first)
    return _shape_batch(lambda i, p: sdb.OrbitBatch(init=i, params=p), w, lo, hi, sample)


def make_model(sdb, w):
    n = w["n"]
    if "model" in w:
        drift, diffusion, nparams = TEMPLATES[w["model"]]
        return sdb.model_from_dsl(w["model"], n, nparams(n), n, drift, diffusion)
    if w["solver"] == "rk4":
        return sdb.ModelSpec(name="kuramoto-ode:%d" % n, nequat=n, nparams=2 * n + 1, nnoise=0,
                             drift=sdb.model._kuramoto_drift)
    return sdb.kuramoto_model(n)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed regions
    (start() / pause() around each; summary() over every sample taken)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, args=(self.proc,), daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self, proc):
        for line in proc.stdout:
            self.lines.append(line.strip())

    def pause(self):
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        self.proc = None

    def summary(self):
        self.pause()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# CPU side: the unmodified reference (baseline/_ref) on a bounded sample

def load_reference():
    """``sdebatch`` installed unmodified into baseline/_ref, or
    None when that install is absent (the oracle port is then timed)."""
    if not os.path.isdir(os.path.join(REF_PATH, "sdebatch")):
        return None
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import sdebatch
    return sdebatch


def cpu_model_name() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _ref_workload(ref, w, m_cpu):
    """The reference's model and the workload's first m_cpu rows, built with
    the reference's own constructors and sampler (model.py:204-277, 291-309)."""
    n = w["n"]
    if "model" in w:
        drift, diffusion, nparams = TEMPLATES[w["model"]]
        model = ref.model_from_dsl(w["model"], n, nparams(n), n, drift, diffusion)
    elif w["solver"] == "rk4":
        model = ref.ModelSpec(name="kuramoto-ode:%d" % n, nequat=n, nparams=2 * n + 1, nnoise=0,
                              drift=ref.model._kuramoto_drift)
    else:
        model = ref.kuramoto_model(n)

    def sample(count, omega, noise, k, first):
        assert first == 0
        return ref.sample_kuramoto_batch(n, count, omega, noise, k, SEED)
    batch = _shape_batch(lambda i, p: ref.OrbitBatch(init=np.ascontiguousarray(i),
                                                     params=np.ascontiguousarray(p)),
                         w, 0, m_cpu, sample)
    return model, batch


def _ref_config(ref, w, m, steps, threads, group):
    # the reference has one noise generator (Philox, rng.py); every other field
    # is the workload's own
    return ref.EngineConfig(dt=w["dt"], tspan=w["dt"] * steps, ksteps=steps, orbits=m,
                            solver=w["solver"], chunk_group=group, seed=SEED, threads=threads,
                            max_store_bytes=1 << 40)


def reference_leg(ref, w, threads, run_seconds: float, repeats: int = 2, warmup: int = 1):
    """One timed leg of the reference: probe the per-orbit-step cost, size a
    sample of M_cpu orbits x S_cpu steps for ~run_seconds per run, pick the
    best chunk_group of {M_cpu, M_cpu/threads, 8192, 512} on a one-step probe,
    then the reference's own bench.time_run (warm-up + timed repeats with a
    store-hash check, bench.py:72-105)."""
    nthreads = (os.cpu_count() or 1) if threads == "all" else threads
    n = w["n"]
    # cost probe: min(M, 256) orbits x 1 step, one group per thread
    m0 = min(w["orbits"], max(nthreads, 256))
    model, batch = _ref_workload(ref, w, m0)
    cfg = _ref_config(ref, w, m0, 1, threads, max(1, m0 // nthreads))
    ref.run_batch(model, cfg, batch)
    t0 = time.perf_counter()
    ref.run_batch(model, cfg, batch)
    per = (time.perf_counter() - t0) / m0  # seconds per orbit-step
    # sample: as many orbits as the budget allows (<= the workload's, <= 2^16,
    # the (G, n, n) drift temporaries <= ~4 GiB), then steps to fill the run
    budget = run_seconds / per
    m_cap = min(w["orbits"], 1 << 16, max(nthreads, int((4 << 30) / (8 * n * n))))
    m_cpu = int(max(min(m0, m_cap), min(m_cap, budget / 2)))
    m_cpu = max(nthreads, m_cpu - m_cpu % nthreads) if m_cpu >= nthreads else m_cpu
    s_cpu = int(max(1, min(w["steps"], budget / m_cpu)))
    model, batch = _ref_workload(ref, w, m_cpu)
    groups = sorted({max(1, min(m_cpu, g)) for g in (m_cpu, m_cpu // nthreads, 8192, 512)})
    probe = {}
    for g in groups:
        cfg = _ref_config(ref, w, m_cpu, 1, threads, g)
        t0 = time.perf_counter()
        ref.run_batch(model, cfg, batch)
        probe[g] = time.perf_counter() - t0
    group = min(probe, key=probe.get)
    cfg = _ref_config(ref, w, m_cpu, s_cpu, threads, group)
    for _ in range(max(0, warmup - 1)):
        ref.run_batch(model, cfg, batch)
    point = ref.bench.time_run(model, cfg, batch, repeats=repeats, warmup=warmup > 0)
    return {"threads": threads, "threads_used": nthreads, "chunk_group": group,
            "chunk_group_probe_s": {str(k): round(v, 4) for k, v in probe.items()},
            "orbits": m_cpu, "steps": s_cpu, "runtimes_s": point.runtimes,
            "value": m_cpu * s_cpu / point.mean, "point": point}


def port_leg(w, threads, run_seconds: float, repeats: int = 2):
    """Fallback when baseline/_ref is absent: the oracle port of run_batch
    (numpy restatement, reference op order, same thread pool)."""
    from oracle import sdeb_oracle as O
    nthreads = (os.cpu_count() or 1) if threads == "all" else threads
    n = w["n"]
    m_cpu = min(w["orbits"], 8192 if n <= 32 else 1024)
    init, params = O.sample_kuramoto_batch(n, m_cpu, (0.2, 0.4), (0.01, 0.03), 0.3, SEED)
    nnoise = 0 if w["solver"] == "rk4" else n
    group = max(1, m_cpu // nthreads)

    def run(steps):
        t0 = time.perf_counter()
        O.integrate(init, params, dt=w["dt"], ksteps=steps, chunks=1, seed=1,
                    solver=w["solver"], nnoise=nnoise, threads=nthreads, group=group)
        return time.perf_counter() - t0
    per = run(2) / 2
    s_cpu = int(max(1, min(w["steps"], run_seconds / per)))
    times = [run(s_cpu) for _ in range(repeats)]
    return {"threads": threads, "threads_used": nthreads, "chunk_group": group,
            "orbits": m_cpu, "steps": s_cpu, "runtimes_s": times,
            "value": m_cpu * s_cpu / float(np.mean(times))}


def cpu_baseline(w, run_seconds: float):
    """threads=1 and threads="all" legs of the reference;
    value = the better leg."""
    ref = load_reference()
    legs = []
    for threads in (1, "all"):
        leg = (reference_leg(ref, w, threads, run_seconds) if ref is not None
               else port_leg(w, threads, run_seconds))
        leg.pop("point", None)
        legs.append(leg)
    best = max(legs, key=lambda l: l["value"])
    return {"value": best["value"], "unit": "orbit-steps/s", "cores": best["threads_used"],
            "kind": "reference" if ref is not None else "port",
            "sample": "%s %s, %d orbits x %d steps of %s, threads=%s, chunk_group=%d "
                      "(best of the thread legs and chunk_group probes), %d host threads "
                      "available (%s)"
                      % ("unmodified sdebatch.run_batch (baseline/_ref) under its own "
                         "bench.time_run" if ref is not None else "oracle port of run_batch",
                         "(Philox: the reference's only generator)", best["orbits"],
                         best["steps"], w["desc"].split(",")[0], best["threads"],
                         best["chunk_group"], os.cpu_count() or 1, cpu_model_name()),
            "legs": legs}


def run_reference_arm(args, w, world, rank):
    """--impl reference: the reference's own CPU path, all host threads, on
    this arm's config and metric; rank 0 alone runs (the others exit)."""
    if rank != 0:
        return
    ref = load_reference()
    total = max(1, args.steps + args.warmup)
    run_seconds = min(args.ref_seconds, max(0.3, 150.0 / total))
    if ref is not None:
        leg = reference_leg(ref, w, "all", run_seconds, repeats=args.steps, warmup=args.warmup)
        point = leg.pop("point")
        times = point.runtimes
        kind = "reference"
        how = ("unmodified sdebatch.run_batch from baseline/_ref through sdebatch.bench.time_run "
               "(%d warm-up, %d timed repeats, store hash checked)" % (args.warmup, args.steps))
    else:
        leg = port_leg(w, "all", run_seconds, repeats=args.steps)
        times = leg["runtimes_s"]
        kind = "port"
        how = "oracle port of run_batch (baseline/_ref absent)"
    ms = 1e3 * float(np.mean(times))
    value = leg["orbits"] * leg["steps"] / (ms * 1e-3)
    line = {
        "impl": "reference", "metric": "orbit-steps/s", "value": value, "unit": "orbit-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (the reference's own sampler, speed/grid presets of the workload)",
        "config": {"workload": args.workload, "headline": w.get("name"), "desc": w["desc"],
                   "n": w["n"], "cpu_sample_orbits": leg["orbits"], "cpu_sample_steps": leg["steps"],
                   "threads": "all", "chunk_group": leg["chunk_group"],
                   "chunk_group_probe_s": leg.get("chunk_group_probe_s")},
        "cpu_baseline": {"value": value, "unit": "orbit-steps/s", "cores": leg["threads_used"],
                         "kind": kind,
                         "sample": "%s; %d orbits x %d SDE steps per bench step, threads=all "
                                   "(%d), chunk_group=%d, %s"
                                   % (how, leg["orbits"], leg["steps"], leg["threads_used"],
                                      leg["chunk_group"], cpu_model_name())},
        "e2e": {"value": value, "unit": "orbit-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# multi-GPU plumbing

def dist_setup(want_gpus: int):
    """torchrun (WORLD_SIZE > 1): one rank per GPU over NCCL; --gpus must
    equal the world size.  Otherwise a single process (which drives --gpus
    devices itself)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        if want_gpus not in (1, world):
            raise SystemExit("--gpus %d but torchrun started %d ranks" % (want_gpus, world))
        import torch
        import torch.distributed as dist_mod
        # SDEB200_BENCH_ONE_GPU=1 (tests only): every rank on GPU 0 over gloo,
        # to exercise the multi-rank bench path on a one-GPU box
        one_gpu = os.environ.get("SDEB200_BENCH_ONE_GPU") == "1"
        if one_gpu:
            local = 0
        # this rank's device is the default context's too (batch sampling,
        # per-step utilities): nothing lands on GPU 0 by accident
        os.environ["SDEB200_DEVICES"] = str(local)
        torch.cuda.set_device(local)
        if one_gpu:
            dist_mod.init_process_group("gloo")
        else:
            dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = dist_mod
    return world, rank, local, dist


def reduce_max(dist, value: float) -> float:
    if dist is None:
        return value
    import torch
    if dist.get_backend() == "gloo":
        return reduce_max_cpu(dist, value)
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_max_cpu(dist, value: float) -> float:
    """Max over ranks on the host (gloo) -- same reduction as reduce_max."""
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def plan_shards(orbits: int, world: int, rank: int, local: int, gpus: int, devices=None):
    """[(device, lo, hi)] this process integrates: its torchrun shard, or one
    shard per device when one process drives --gpus devices (``devices``
    overrides the ids, e.g. 0,0,0,0 to exercise N shards on one GPU)."""
    from paper_1908_03869_b200.engine import shard_bounds
    if world > 1:
        return [(local,) + shard_bounds(orbits, world, rank)]
    devs = list(devices) if devices else list(range(gpus))
    return [(d,) + shard_bounds(orbits, len(devs), g) for g, d in enumerate(devs)]


# ---------------------------------------------------------------------------
# GPU side

def measure(args, name, w, shards, world, dist, clocks, e2e_steps, peak_ops):
    """Device-resident and end-to-end orbit-steps/s of one workload over
    ``shards`` (this process's (device, lo, hi) list)."""
    import torch

    import paper_1908_03869_b200 as sdb
    from paper_1908_03869_b200 import _native as nat
    from paper_1908_03869_b200.engine import make_desc

    if w.get("model") == "kuramoto_template":
        os.environ["SDEB200_NO_NATIVE_KURAMOTO"] = "1"  # the generated program, not the stepper
    else:
        os.environ.pop("SDEB200_NO_NATIVE_KURAMOTO", None)
    n, m_total, steps = w["n"], w["orbits"], w["steps"]
    chunks = steps // w["ksteps"]
    coherence = bool(w.get("coherence"))
    model = make_model(sdb, w)
    devices = tuple(d for d, _, _ in shards)
    lib = nat.lib()
    program_handle = None
    if "model" in w:
        from paper_1908_03869_b200 import program
        program_handle = program.model_program(model).handle

    legs = []
    for dev, lo, hi in shards:
        torch.cuda.set_device(dev)
        rows = hi - lo
        batch = make_batch(sdb, w, lo, hi)
        cfg = sdb.EngineConfig(dt=w["dt"], tspan=w["dt"] * steps, ksteps=w["ksteps"], orbits=rows,
                               solver=w["solver"], seed=SEED, stream=w["stream"],
                               coupling=args.coupling, devices=(dev,), max_store_bytes=1 << 40)
        assert sdb.iteration_count(cfg.tspan, cfg.dt, cfg.ksteps) == chunks
        leg = dict(dev=dev, lo=lo, hi=hi, rows=rows, batch=batch, ctx=nat.context((dev,)),
                   desc=make_desc(model, cfg, chunks, rows, orbit_offset=lo),
                   init=torch.from_numpy(np.ascontiguousarray(batch.init)).cuda(dev),
                   params=torch.from_numpy(np.ascontiguousarray(batch.params)).cuda(dev),
                   values=(torch.empty((rows, 2, chunks + 1), dtype=torch.float64, device=dev)
                           if coherence else
                           torch.empty((rows, chunks, n), dtype=torch.float64, device=dev)),
                   fail=torch.empty(rows, dtype=torch.int64, device=dev),
                   flush=torch.empty(512 << 20, dtype=torch.uint8, device=dev),
                   stream=torch.cuda.current_stream(dev))
        legs.append(leg)

    def launch(leg):
        torch.cuda.set_device(leg["dev"])
        ctx, desc, st = leg["ctx"], leg["desc"], leg["stream"].cuda_stream
        ptrs = (leg["init"].data_ptr(), leg["params"].data_ptr(), leg["values"].data_ptr(),
                leg["fail"].data_ptr())
        if coherence:
            nat.check(lib.sdb_run_coherence_device(ctx, desc, *ptrs, st), ctx,
                      "sdb_run_coherence_device")
        elif program_handle is not None:
            nat.check(lib.sdb_run_model_device(ctx, program_handle, desc, *ptrs, st), ctx,
                      "sdb_run_model_device")
        else:
            nat.check(lib.sdb_run_device(ctx, desc, *ptrs, st), ctx, "sdb_run_device")

    def sync_all():
        for leg in legs:
            torch.cuda.synchronize(leg["dev"])

    # warm-up (the first call per shape also picks the lane layout)
    for _ in range(max(args.warmup, 3)):
        for leg in legs:
            launch(leg)
    sync_all()
    import ctypes
    lay = [ctypes.c_int32() for _ in range(5)]
    lib.sdb_last_layout(legs[0]["ctx"], *(ctypes.byref(v) for v in lay))
    lanes, persistent, ctas_per_sm, variant, _ = (int(v.value) for v in lay)
    lane_width = int(lib.sdb_last_lane_width(legs[0]["ctx"]))
    launches_per_step = sum(int(lib.sdb_last_launch_count(l["ctx"])) for l in legs)

    for leg in legs:
        torch.cuda.set_device(leg["dev"])
        leg["ev"] = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                     for _ in range(args.steps)]
    barrier(dist)
    sync_all()
    clocks.start()
    time.sleep(0.15)  # let the sampler attach before the first timed launch
    for i in range(args.steps):
        for leg in legs:
            torch.cuda.set_device(leg["dev"])
            leg["flush"].zero_()
            leg["ev"][i][0].record(leg["stream"])
            launch(leg)
            leg["ev"][i][1].record(leg["stream"])
    sync_all()
    clocks.pause()
    barrier(dist)
    per_leg = [[a.elapsed_time(b) for a, b in leg["ev"]] for leg in legs]
    kernel_ms = [max(col) for col in zip(*per_leg)]  # the step ends with its slowest GPU
    ms_per_step = reduce_max(dist, float(sum(kernel_ms))) / args.steps
    orbit_steps = float(m_total) * steps
    value = orbit_steps / (ms_per_step * 1e-3)
    for leg in legs:
        assert torch.isfinite(leg["values"]).all().item(), "non-finite states in the bench run"

    # --- e2e through the public API (host numpy buffers) ---
    api = sdb.run_coherence if coherence else sdb.run_batch
    if len(legs) == 1:
        host = legs[0]["batch"]
        lo0, rows_e2e = legs[0]["lo"], legs[0]["rows"]
    else:  # one process, N devices: the whole batch through EngineConfig(devices=range(N))
        host = sdb.OrbitBatch(init=np.concatenate([l["batch"].init for l in legs]),
                              params=np.concatenate([l["batch"].params for l in legs]))
        lo0, rows_e2e = legs[0]["lo"], legs[-1]["hi"] - legs[0]["lo"]
    cfg_e2e = sdb.EngineConfig(dt=w["dt"], tspan=w["dt"] * steps, ksteps=w["ksteps"],
                               orbits=rows_e2e, solver=w["solver"], seed=SEED, stream=w["stream"],
                               coupling=args.coupling, devices=devices, max_store_bytes=1 << 40)
    for leg in legs:  # the device-resident copies are not needed any more
        for key in ("init", "params", "values", "fail", "flush"):
            leg.pop(key)
        leg.pop("batch")
    gc.collect()
    torch.cuda.empty_cache()
    def e2e_leg(batch_h, steps_h):
        api(model, cfg_e2e, batch_h, orbit_offset=lo0)  # warm: layout cache, staging slots
        barrier(dist)
        per_call, hashes = [], []
        for _ in range(steps_h):
            t0 = time.perf_counter()
            store = api(model, cfg_e2e, batch_h, orbit_offset=lo0)
            per_call.append(time.perf_counter() - t0)
            # repeat-determinism check (the reference bench hashes every repeat,
            # bench.py:91-96) outside the per-call timing; the store is then
            # dropped, as a sweep that consumes each result would
            hashes.append(result_hash(sdb, store, coherence))
            del store
        return reduce_max(dist, float(np.mean(per_call))), per_call, hashes

    # the contract's e2e: inputs from pinned host memory (sdb.pin_batch, filled
    # outside the timed region like the reference bench's batch sampling); the
    # store is the ordinary pageable array run_batch returns
    pinned = sdb.pin_batch(host)
    e2e_s, per_call, hashes = e2e_leg(pinned, e2e_steps)
    del pinned
    # the same with ordinary pageable numpy inputs (the library stages them)
    e2e_pg, _, hashes_pg = e2e_leg(host, max(1, min(e2e_steps, 3)))
    h2d = host.init.nbytes + host.params.nbytes
    d2h = (rows_e2e * (chunks + 1) * 2 * 8 if coherence else rows_e2e * chunks * n * 8) + rows_e2e * 8
    e2e = {"value": orbit_steps / e2e_s, "unit": "orbit-steps/s",
           "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
           "ms_per_step": e2e_s * 1e3, "median_ms": float(np.median(per_call)) * 1e3,
           "host_buffers": "inputs in pinned host memory (sdb.pin_batch), store: the pageable "
                           "numpy array %s returns (large stores on recycled host mappings)"
                           % api.__name__,
           "pageable_inputs": {"value": orbit_steps / e2e_pg, "ms_per_step": e2e_pg * 1e3},
           "result_sha256": hashes[0][:16],
           "repeats_identical": len(set(hashes + hashes_pg)) == 1}
    del host
    gc.collect()

    # --- roofline (FP64 pipe) of the stepper on the first device ---
    ops = (template_fp64_ops(n, w["model"], args.coupling) if "model" in w
           else algorithmic_fp64_ops(n, w["solver"], args.coupling))
    leg_ms = float(np.mean(per_leg[0]))
    leg_orbit_steps = float(legs[0]["rows"]) * steps
    achieved = ops * leg_orbit_steps / (leg_ms * 1e-3)
    roofline = {
        "bound": "fp64", "unit": "TFLOP/s",
        "achieved": 2 * achieved / 1e12, "peak": 2 * peak_ops / 1e12,
        "frac": achieved / peak_ops,
        "frac_basis": "the kernel's own algorithmic FP64 lane-ops per orbit-step (%s form)"
                      % ("generated template program" if "model" in w else args.coupling),
        "algorithmic_fp64_ops_per_orbit_step": ops,
        "traffic": measured_traffic(name),
        "traffic_basis": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch "
                         "(profiles/traffic.json)",
        "algorithmic_bytes_per_launch": algorithmic_bytes(w, legs[0]["rows"]),
        "achieved_hbm_gbs": algorithmic_bytes(w, legs[0]["rows"]) / (leg_ms * 1e-3) / 1e9,
        "peak_source": "measured live: sdb_fp64_peak DFMA-throughput kernel (FLOP = 2 x DFMA)",
    }
    if w["solver"] == "em" and "model" not in w:
        roofline["w_em_ops_per_orbit_step"] = pairwise_equivalent_ops(n)
        roofline["w_em_frac"] = (pairwise_equivalent_ops(n) * leg_orbit_steps
                                 / (leg_ms * 1e-3) / peak_ops)
        roofline["w_em_basis"] = ("SURVEY.md 8d W_EM(n) = 9n(n-1)+41n of the reference's "
                                  "term-by-term algorithm against the same time; exceeds 1 for "
                                  "the meanfield form, which does O(n) instead of O(n^2) work")
    return {
        "name": name, "value": value, "ms_per_step": ms_per_step, "kernel_ms": kernel_ms,
        "e2e": e2e, "roofline": roofline, "launches_per_step": launches_per_step,
        "layout": {"lanes_per_orbit": lanes, "oscillators_per_lane": lane_width,
                   "persistent_grid": bool(persistent), "ctas_per_sm": ctas_per_sm,
                   "register_capped": bool(variant)},
        "orbits_per_gpu": [l["rows"] for l in legs],
    }


def algorithmic_bytes(w, rows: int) -> float:
    """HBM bytes one launch must move: init + params read once, the samples
    1..k (or (r, Phi) planes) and the failure word written once."""
    n, chunks = w["n"], w["steps"] // w["ksteps"]
    nparams = TEMPLATES[w["model"]][2](n) if "model" in w else 2 * n + 1
    out = 2 * (chunks + 1) if w.get("coherence") else chunks * n
    return float(rows) * 8.0 * (n + nparams + out + 1)


def cold_probe(args):
    """--cold-probe: in a fresh process, the first run_batch call after the
    batch exists (its sampling touched the device, so CUDA context creation
    is outside), then a second call: prints both."""
    import paper_1908_03869_b200 as sdb
    w = WORKLOADS[args.workload]
    model = make_model(sdb, w)
    devices = tuple(range(args.gpus))
    batch = make_batch(sdb, w)
    cfg = sdb.EngineConfig(dt=w["dt"], tspan=w["dt"] * w["steps"], ksteps=w["ksteps"],
                           orbits=w["orbits"], solver=w["solver"], seed=SEED, stream=w["stream"],
                           coupling=args.coupling, devices=devices, max_store_bytes=1 << 40)
    api = sdb.run_coherence if w.get("coherence") else sdb.run_batch
    times = []
    for _ in range(2):
        t0 = time.perf_counter()
        store = api(model, cfg, batch)
        times.append(time.perf_counter() - t0)
        del store
        gc.collect()
    print(json.dumps({"cold_s": times[0], "second_s": times[1]}), flush=True)


def run_cold(args, name, w):
    """cold_e2e of one workload: bench.py --cold-probe in a subprocess with an
    empty on-disk layout cache (a fresh box)."""
    with tempfile.TemporaryDirectory() as tmp:
        env = dict(os.environ, SDEB200_TUNE_CACHE=os.path.join(tmp, "layouts.json"))
        env.pop("SDEB200_TUNE", None)  # the default, budgeted search of a first call
        out = subprocess.run([sys.executable, os.path.abspath(__file__), "--cold-probe",
                              "--workload", name, "--gpus", str(args.gpus), "--coupling",
                              args.coupling], capture_output=True, text=True, env=env,
                             timeout=900)
    if out.returncode != 0:
        return {"error": (out.stderr or out.stdout).strip().splitlines()[-1:]}
    res = json.loads(out.stdout.strip().splitlines()[-1])
    orbit_steps = float(w["orbits"]) * w["steps"]
    return {"value": orbit_steps / res["cold_s"], "unit": "orbit-steps/s",
            "ms": res["cold_s"] * 1e3, "second_call_ms": res["second_s"] * 1e3,
            "how": "first run_batch() of a fresh process (empty layout cache; batch sampling "
                   "and CUDA context creation before the timed call), host buffers"}


def run_ours(args, world, rank, local, dist):
    # the measured process amortises a complete layout search in its warm-up
    # (SDEB200_TUNE=thorough); the cold_e2e subprocess runs the default,
    # budgeted search a first call pays
    os.environ.setdefault("SDEB200_TUNE", "thorough")
    # and keeps its decisions to itself: no timing depends on ~/.cache
    os.environ.setdefault("SDEB200_TUNE_CACHE", os.path.join(
        tempfile.mkdtemp(prefix="sdeb200-bench-"), "layouts.tsv"))
    import torch

    from paper_1908_03869_b200 import _native as nat

    w_top = WORKLOADS[args.workload]
    names = list(w_top.get("sizes", (args.workload,)))
    headline = w_top.get("headline", args.workload)
    secondary = list(w_top.get("secondary", ())) if not args.no_secondary else []
    if world == 1:
        have = nat.device_count()
        if args.gpus > have:
            raise SystemExit("--gpus %d but only %d CUDA device(s) are visible" % (args.gpus, have))
        if args.devices and (max(args.devices) >= have or len(set(args.devices)) != args.gpus):
            raise SystemExit("--devices %s does not name --gpus %d distinct visible devices"
                             % (args.devices, args.gpus))
    n_gpus = world if world > 1 else args.gpus
    torch.cuda.set_device(local)
    # the cold first call runs first, in its own process, before this one has
    # filled host memory with batches, pinned staging and recycled stores
    cold = None
    if rank == 0 and world == 1 and not args.no_cold:
        cold = run_cold(args, headline, WORKLOADS[headline])
    peak_ops = ctypes_peak(nat.lib(), nat.context((local,)))
    clocks = ClockSampler(local)
    results = {}
    for name in names + secondary:
        w = WORKLOADS[name]
        shards = plan_shards(w["orbits"], world, rank, local, args.gpus, args.devices)
        e2e_steps = max(1, min(args.steps, 5 if name in names else 3))
        results[name] = measure(args, name, w, shards, world, dist, clocks, e2e_steps, peak_ops)
        gc.collect()
        torch.cuda.empty_cache()
    clock_info = clocks.summary()
    head = results[headline]
    wh = WORKLOADS[headline]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wh, args.cpu_seconds)

    if rank != 0:
        return

    def brief(r):
        out = {"value": r["value"], "ms_per_step": r["ms_per_step"], "e2e": r["e2e"]["value"],
               "e2e_ms": r["e2e"]["ms_per_step"], "frac": r["roofline"]["frac"],
               "w_em_frac": r["roofline"].get("w_em_frac"),
               "traffic": r["roofline"]["traffic"],
               "achieved_hbm_gbs": r["roofline"]["achieved_hbm_gbs"]}
        out.update(r["layout"])
        return out

    line = {
        "metric": "orbit-steps/s", "value": head["value"], "unit": "orbit-steps/s",
        "n_gpus": n_gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        # only the paper-protocol workloads have a published number (SODECL on a
        # P100); cfg3 has none
        "vs_baseline": (head["value"] / wh["published"]) if wh.get("published") else None,
        "dtype": "f64",
        "data": "synthetic (device-sampled Kuramoto batch, reference sampler bit-exact)",
        "config": {"workload": args.workload, "headline": headline, "desc": w_top["desc"],
                   "n": wh["n"], "orbits": wh["orbits"], "sde_steps": wh["steps"],
                   "ksteps": wh["ksteps"], "solver": wh["solver"], "stream": wh["stream"],
                   "coupling": args.coupling, "orbits_per_gpu": head["orbits_per_gpu"],
                   "template_model": wh.get("model"),
                   "parallelism": "contiguous orbit shards x%d (%s), no data-path collective"
                                  % (len(head["orbits_per_gpu"]) * world,
                                     "torchrun, one process per GPU" if world > 1
                                     else "one process driving devices %s"
                                     % (args.devices or list(range(args.gpus)))),
                   "l2": "flushed (512 MiB memset) between timed steps, outside the event "
                         "pairs; inputs also exceed L2 for cfg3",
                   **head["layout"]},
        "e2e": head["e2e"], "cold_e2e": cold, "roofline": head["roofline"],
        "cpu_baseline": cpu,
        "gpu_launches": head["launches_per_step"] * args.steps * world,
        "clocks": clock_info,
        "kernel_ms": head["kernel_ms"],
        "sizes": {k: brief(results[k]) for k in names},
        "secondary": {k: brief(results[k]) for k in secondary},
    }
    print(json.dumps(line), flush=True)


def result_hash(sdb, store, coherence: bool) -> str:
    """SHA-256 of one e2e result: the store (storage.store_hash) or, for the
    fused coherence run, its r / Phi series."""
    if not coherence:
        return sdb.store_hash(store)
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(store.r, dtype="<f8").tobytes())
    h.update(np.ascontiguousarray(store.phi, dtype="<f8").tobytes())
    return h.hexdigest()


def ctypes_peak(lib, ctx) -> float:
    import ctypes
    ops = ctypes.c_double()
    ms = ctypes.c_double()
    from paper_1908_03869_b200 import _native as nat
    nat.check(lib.sdb_fp64_peak(ctx, ctypes.byref(ops), ctypes.byref(ms)), ctx, "sdb_fp64_peak")
    return ops.value


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=DEFAULT_WORKLOAD)
    ap.add_argument("--coupling", choices=["meanfield", "pairwise"], default="meanfield")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cold", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=4.0,
                    help="seconds per timed reference run in the cpu_baseline legs")
    ap.add_argument("--ref-seconds", type=float, default=8.0,
                    help="cap on the seconds per step of --impl reference")
    ap.add_argument("--devices", type=lambda t: [int(x) for x in t.split(",")], default=None,
                    help="device id per in-process shard (default 0..gpus-1); repeats run "
                         "several shards on one GPU (host-pipeline studies)")
    ap.add_argument("--cold-probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.cold_probe:
        cold_probe(args)
        return
    w = WORKLOADS[args.workload]
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        head = w.get("headline", args.workload)
        run_reference_arm(args, dict(WORKLOADS[head], name=head), world, rank)
        return
    world, rank, local, dist = dist_setup(args.gpus)
    try:
        run_ours(args, world, rank, local, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
