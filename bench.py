#!/usr/bin/env python
"""Benchmark: orbit-steps/s of stochastic Kuramoto Euler-Maruyama on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2] [--coupling meanfield|pairwise]

One "step" = one complete run of the workload (all orbits x all SDE steps)
through the fused kernel.  Default workload = BASELINE.json configs[1]
(cfg2): n=16, 65,536 orbits over a 256 K x 256 sigma grid, sfc64 streams,
dt=1e-3, 10^4 steps, final state only.  Multi-GPU (torchrun): each rank
integrates its own 65,536-orbit shard with global orbit ids
[rank*M, (rank+1)*M) -- weak scaling, no data-path collective (the path is
embarrassingly parallel); timing is max over ranks.

  value    device-resident inputs (sdb_run_device), CUDA events around each
           kernel launch, L2 flushed (512 MiB memset) between timed steps
           outside the event pairs.
  e2e      the public API run_batch() with numpy host buffers: H2D of
           init/params and D2H of the store inside every timed step.
  roofline FP64 pipe: algorithmic FP64 lane-ops of the kernel's algorithm
            / kernel time, against the FP64 DFMA peak
           measured live (sdb_fp64_peak; MEASURED_PEAKS.json has no FP64 figure).
  cpu_baseline  the oracle port (numpy restatement of the reference's
           run_batch, same op order, same thread pool) on a bounded sample.
--impl reference times that CPU implementation alone (rank 0).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")

WORKLOADS = {
    # BASELINE.json configs[1] -- the headline
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

def make_batch(sdb, w, orbit_offset: int, seed: int = 20260809):
    n, m = w["n"], w["orbits"]
    local = np.arange(m)
    if w["batch"] == "speed":
        return sdb.sample_kuramoto_batch(n, m, (0.01, 0.03), (0.001, 0.003), 1.0, seed,
                                         orbit_offset=orbit_offset)
    if w["batch"] == "kgrid":
        b = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.03), 0.0, seed,
                                      orbit_offset=orbit_offset)
        params = b.params.copy()
        params[:, 0] = np.linspace(0.0, 0.5, 256)[(local // 256) % 256]
        params[:, n + 1:] = np.geomspace(1e-3, 1e-1, 256)[local % 256][:, None]
        return sdb.OrbitBatch(init=b.init, params=params)
    if w["batch"] == "kgrid_ode":  # cfg4: 512 K x 512 omega draws, zero diffusion
        b = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.0, 0.0), 0.0, seed,
                                      orbit_offset=orbit_offset)
        params = b.params.copy()
        params[:, 0] = np.linspace(0.0, 2.0, 512)[(local // 512) % 512]
        return sdb.OrbitBatch(init=b.init, params=params)
    if w["batch"] == "resample":  # cfg5: 512 sets x 256 realisations
        sets = m // 256
        b = sdb.sample_kuramoto_batch(n, sets, (0.2, 0.4), (0.01, 0.03), 0.0, seed,
                                      orbit_offset=orbit_offset // 256)
        params = b.params.copy()
        params[:, 0] = np.linspace(0.05, 0.8, 16)[np.arange(sets) % 16]
        return sdb.OrbitBatch(init=np.repeat(b.init, 256, axis=0),
                              params=np.repeat(params, 256, axis=0))
    if w["batch"] == "uniform":  # generic template models: seeded uniform draws
        g = np.random.default_rng(seed + orbit_offset)
        nparams = TEMPLATES[w["model"]][2](n)
        return sdb.OrbitBatch(init=g.uniform(-1.0, 1.0, (m, n)),
                              params=g.uniform(0.05, 0.5, (m, nparams)))
    raise ValueError(w["batch"])


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
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

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
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
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


def dist_setup(want_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist_mod
        torch.cuda.set_device(local)
        dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = dist_mod
    return world, rank, local, dist


def reduce_max(dist, value: float) -> float:
    if dist is None:
        return value
    import torch
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


# ---------------------------------------------------------------------------
# CPU side: the oracle port (reference algorithm) on a bounded sample

def cpu_sample_rate(w, seconds: float, threads: int, stream_override=None):
    """orbit-steps/s of the oracle port (numpy restatement of the reference's
    run_batch, engine.py:184-277) on M_cpu orbits x S_cpu steps of workload w."""
    from oracle import sdeb_oracle as O
    n = w["n"]
    m_cpu = min(w["orbits"], 8192 if n <= 32 else 1024)
    init, params = O.sample_kuramoto_batch(n, m_cpu, (0.2, 0.4), (0.01, 0.03), 0.3, 20260809)
    if w["solver"] == "rk4":
        params[:, n + 1:] = 0.0
    stream = stream_override or w["stream"]
    group = max(1, m_cpu // threads)
    nnoise = 0 if w["solver"] == "rk4" else n
    fns = {}
    if "model" in w:  # the reference's interpreter, restated (oracle.expression_model)
        drift_t, diffusion_t, nparams = TEMPLATES[w["model"]]
        fns = dict(zip(("drift", "diffusion"), O.expression_model(drift_t, diffusion_t)))
        g = np.random.default_rng(1)
        params = g.uniform(0.05, 0.5, (m_cpu, nparams(n)))

    def run(steps):
        t0 = time.perf_counter()
        O.integrate(init, params, dt=w["dt"], ksteps=steps, chunks=1, seed=1,
                    solver=w["solver"], nnoise=nnoise, stream=stream, threads=threads, group=group,
                    **fns)
        return time.perf_counter() - t0

    probe = 3
    dt_probe = run(probe)
    s_cpu = int(max(probe, min(100000, seconds / max(dt_probe / probe, 1e-9))))
    return m_cpu, s_cpu, group, run


def cpu_baseline(w, seconds: float):
    threads = os.cpu_count() or 1
    m_cpu, s_cpu, group, run = cpu_sample_rate(w, seconds, threads, "philox")
    elapsed = run(s_cpu)
    return {"value": m_cpu * s_cpu / elapsed, "unit": "orbit-steps/s", "cores": threads,
            "kind": "port",
            "sample": "oracle port of run_batch (numpy, reference op order, %s stream), "
                      "%d orbits x %d steps of %s, ThreadPool(%d) over groups of %d, %.1f s"
                      % ("philox (the reference's own generator)" if w["solver"] == "em" else "no", m_cpu, s_cpu,
                         w["desc"].split(",")[0], threads, group, elapsed)}


def run_reference_arm(args, w, world, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    m_cpu, s_cpu, group, run = cpu_sample_rate(w, args.ref_seconds, threads, "philox")
    for _ in range(args.warmup):
        run(max(1, s_cpu // 10))
    times = [run(s_cpu) for _ in range(args.steps)]
    ms = 1e3 * float(np.mean(times))
    value = m_cpu * s_cpu / (ms * 1e-3)
    line = {
        "impl": "reference", "metric": "orbit-steps/s", "value": value, "unit": "orbit-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (sampled batch, reference sampler)",
        "config": {"workload": args.workload, "desc": w["desc"], "n": w["n"],
                   "cpu_sample_orbits": m_cpu, "cpu_sample_steps": s_cpu},
        "cpu_baseline": {"value": value, "unit": "orbit-steps/s", "cores": threads,
                         "kind": "port",
                         "sample": "%d orbits x %d SDE steps per bench step, oracle port of "
                                   "run_batch (reference is pure Python: no compiled _ref), "
                                   "ThreadPool(%d) over groups of %d" % (m_cpu, s_cpu, threads,
                                                                         group)},
        "e2e": {"value": value, "unit": "orbit-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

def run_ours(args, w, world, rank, local, dist):
    import torch

    import paper_1908_03869_b200 as sdb
    from paper_1908_03869_b200 import _native as nat
    from paper_1908_03869_b200.engine import make_desc

    torch.cuda.set_device(local)
    if w.get("model") == "kuramoto_template":
        os.environ["SDEB200_NO_NATIVE_KURAMOTO"] = "1"  # the generated program, not the stepper
    n, m, steps = w["n"], w["orbits"], w["steps"]
    chunks = steps // w["ksteps"]
    model = make_model(sdb, w)
    offset = rank * m
    batch = make_batch(sdb, w, offset)
    cfg = sdb.EngineConfig(dt=w["dt"], tspan=w["dt"] * steps, ksteps=w["ksteps"], orbits=m,
                           solver=w["solver"], seed=20260809, stream=w["stream"],
                           coupling=args.coupling, devices=(local,),
                           max_store_bytes=1 << 40)
    assert sdb.iteration_count(cfg.tspan, cfg.dt, cfg.ksteps) == chunks
    ctx = nat.context((local,))
    lib = nat.lib()
    desc = make_desc(model, cfg, chunks, m, orbit_offset=offset)

    d_init = torch.from_numpy(np.ascontiguousarray(batch.init)).cuda()
    d_params = torch.from_numpy(np.ascontiguousarray(batch.params)).cuda()
    coherence = bool(w.get("coherence"))
    d_values = (torch.empty((m, 2, chunks + 1), dtype=torch.float64, device="cuda") if coherence
                else torch.empty((m, chunks, n), dtype=torch.float64, device="cuda"))
    d_fail = torch.empty(m, dtype=torch.int64, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    program_handle = None
    if desc.model == nat.SDB_MODEL_EXPRESSION:
        from paper_1908_03869_b200 import program
        program_handle = program.model_program(model).handle

    def launch():
        if coherence:
            nat.check(lib.sdb_run_coherence_device(ctx, desc, d_init.data_ptr(),
                                                   d_params.data_ptr(), d_values.data_ptr(),
                                                   d_fail.data_ptr(), stream.cuda_stream),
                      ctx, "sdb_run_coherence_device")
            return
        if program_handle is not None:
            nat.check(lib.sdb_run_model_device(ctx, program_handle, desc, d_init.data_ptr(),
                                               d_params.data_ptr(), d_values.data_ptr(),
                                               d_fail.data_ptr(), stream.cuda_stream),
                      ctx, "sdb_run_model_device")
            return
        nat.check(lib.sdb_run_device(ctx, desc, d_init.data_ptr(), d_params.data_ptr(),
                                     d_values.data_ptr(), d_fail.data_ptr(), stream.cuda_stream),
                  ctx, "sdb_run_device")

    for _ in range(max(args.warmup, 3)):
        launch()
    torch.cuda.synchronize()
    import ctypes
    lay = [ctypes.c_int32() for _ in range(5)]
    lib.sdb_last_layout(ctx, *(ctypes.byref(v) for v in lay))
    lanes, persistent, ctas_per_sm, variant, _ = (int(v.value) for v in lay)
    lane_width = int(lib.sdb_last_lane_width(ctx))
    launches_per_step = int(lib.sdb_last_launch_count(ctx))

    clocks = ClockSampler(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    barrier(dist)
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)  # let the sampler attach before the first timed launch
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        launch()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    barrier(dist)
    clock_info = clocks.stop()
    kernel_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = reduce_max(dist, float(sum(kernel_ms)))
    ms_per_step = total_ms / args.steps
    orbit_steps = float(m) * steps
    value = world * orbit_steps / (ms_per_step * 1e-3)

    # sanity: the timed runs produced finite final states
    assert torch.isfinite(d_values).all().item(), "non-finite states in the benchmark run"

    # --- e2e through the public API (host numpy buffers) ---
    host_batch = sdb.OrbitBatch(init=batch.init.copy(), params=batch.params.copy())
    api = sdb.run_coherence if coherence else sdb.run_batch
    api(model, cfg, host_batch, orbit_offset=offset)  # warm (autotune cache, pinned staging)
    barrier(dist)
    e2e_steps = max(1, min(args.steps, 5))
    per_call, hashes = [], []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        store = api(model, cfg, host_batch, orbit_offset=offset)
        per_call.append(time.perf_counter() - t0)
        # repeat-determinism check (the reference bench hashes every repeat,
        # bench.py:91-96) outside the per-call timing; the store is then
        # dropped, as a sweep that consumes each result would
        hashes.append(result_hash(sdb, store, coherence))
        del store
    e2e_s = reduce_max(dist, float(sum(per_call))) / e2e_steps
    h2d = batch.init.nbytes + batch.params.nbytes
    d2h = (m * (chunks + 1) * 2 * 8 if coherence else m * chunks * n * 8) + m * 8
    e2e = {"value": world * orbit_steps / e2e_s, "unit": "orbit-steps/s",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "ms_per_step": e2e_s * 1e3,
           "median_ms": float(np.median(per_call)) * 1e3,
           "host_buffers": "pageable numpy (%s; large stores on recycled host mappings)"
                           % api.__name__,
           "result_sha256": hashes[0][:16],
           "repeats_identical": len(set(hashes)) == 1}

    # --- roofline (FP64 pipe) ---
    peak_ops = ctypes_peak(lib, ctx)
    ops = (template_fp64_ops(n, w["model"], args.coupling) if "model" in w
           else algorithmic_fp64_ops(n, w["solver"], args.coupling))
    achieved = ops * orbit_steps / (np.mean(kernel_ms) * 1e-3)
    roofline = {
        "bound": "fp64", "unit": "TFLOP/s",
        "achieved": 2 * achieved / 1e12, "peak": 2 * peak_ops / 1e12,
        "frac": achieved / peak_ops,
        "traffic": measured_traffic(args.workload),
        "algorithmic_fp64_ops_per_orbit_step": ops,
        "peak_source": "measured live: sdb_fp64_peak DFMA-throughput kernel (FLOP = 2 x DFMA)",
        "pairwise_equivalent_frac": pairwise_equivalent_ops(n) * orbit_steps
        / (np.mean(kernel_ms) * 1e-3) / peak_ops if w["solver"] == "em" else None,
    }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": "orbit-steps/s", "value": value, "unit": "orbit-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak",
            # only the paper-protocol workloads have a published number (SODECL on a
            # P100); cfg2 has none
            "vs_baseline": (value / w["published"]) if w.get("published") else None,
            "dtype": "f64",
            "data": "synthetic (device-sampled Kuramoto batch, reference sampler bit-exact)",
            "config": {"workload": args.workload, "desc": w["desc"], "n": n,
                       "orbits_per_gpu": m, "sde_steps": steps, "ksteps": w["ksteps"],
                       "solver": w["solver"], "stream": w["stream"], "coupling": args.coupling,
                       "lanes_per_orbit": lanes, "oscillators_per_lane": lane_width,
                       "persistent_grid": bool(persistent),
                       "ctas_per_sm": ctas_per_sm, "register_capped": bool(variant),
                       "template_model": w.get("model"),
                       "parallelism": "orbit-shard x%d" % world,
                       "l2": "flushed (512 MiB memset) between timed steps, outside the "
                             "event pairs"},
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clock_info,
            "kernel_ms": kernel_ms,
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
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2")
    ap.add_argument("--coupling", choices=["meanfield", "pairwise"], default="meanfield")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-seconds", type=float, default=2.0)
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    world, rank, local, dist = (int(os.environ.get("WORLD_SIZE", "1")),
                                int(os.environ.get("RANK", "0")),
                                int(os.environ.get("LOCAL_RANK", "0")), None)
    if args.impl == "reference":
        run_reference_arm(args, w, world, rank)
        return
    world, rank, local, dist = dist_setup(args.gpus)
    try:
        run_ours(args, w, world, rank, local, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
