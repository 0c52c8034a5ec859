"""numpy restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.

Restates, in the same operation order, what the reference package ``sdebatch``
computes on the path ``run_batch -> normals_for_orbits -> euler_maruyama_step
-> _kuramoto_drift``.  Every function cites the
reference ``file:line`` it follows (paths relative to
``/root/reference/pkg/src/sdebatch``).  The one generalisation over the
reference is ``integrate(..., orbit_ids=...)``: explicit global orbit ids, so
an arbitrary shard (orbits that do not start at 0) can be checked; with
``orbit_ids = arange(M)`` it is bit-identical to ``run_batch``
(tests/test_oracle.py checks that against the golden stores).

The sfc64 / xoshiro256++ / SplitMix64 streams are NOT in the reference; they
restate the published algorithms and the stream layout defined in DESIGN.md
("Noise streams").  Parity for them is pinned against numpy's SFC64 and a
hand-derived xoshiro256++ KAT, not against the reference.

Imported only by tests/, __graft_entry__.smoke() and bench.py (CPU baseline).
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# rng.py:31-45
PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85
PHILOX_ROUNDS = 10
MASK32 = 0xFFFFFFFF
MASK64 = 0xFFFFFFFFFFFFFFFF
SAMPLING_TAG = 0xFFFFFFFF
TWO_NEG_32 = 2.0 ** -32
TWO_PI = 2.0 * math.pi

STREAMS = ("philox", "sfc64", "xoshiro256pp")


# ---------------------------------------------------------------------------
# Philox-4x32-10 (rng.py:74-118)

def philox_block(counter, key):
    """Scalar Philox-4x32-10; rng.py:74-90."""
    x0, x1, x2, x3 = counter
    k0, k1 = key
    for _ in range(PHILOX_ROUNDS):
        p0 = PHILOX_M0 * x0
        p1 = PHILOX_M1 * x2
        x0, x1, x2, x3 = (((p1 >> 32) ^ x1 ^ k0) & MASK32, p1 & MASK32,
                          ((p0 >> 32) ^ x3 ^ k1) & MASK32, p0 & MASK32)
        k0 = (k0 + PHILOX_W0) & MASK32
        k1 = (k1 + PHILOX_W1) & MASK32
    return (x0, x1, x2, x3)


def philox_words(k0, k1, c0, c1, c2, c3):
    """Vectorised Philox-4x32-10 over broadcast uint32 arrays; rng.py:93-118."""
    k0 = np.asarray(k0, dtype=np.uint32)
    k1 = np.asarray(k1, dtype=np.uint32)
    x0 = np.asarray(c0, dtype=np.uint32)
    x1 = np.asarray(c1, dtype=np.uint32)
    x2 = np.asarray(c2, dtype=np.uint32)
    x3 = np.asarray(c3, dtype=np.uint32)
    m0, m1 = np.uint64(PHILOX_M0), np.uint64(PHILOX_M1)
    w0, w1 = np.uint32(PHILOX_W0), np.uint32(PHILOX_W1)
    sh = np.uint64(32)
    with np.errstate(over="ignore"):
        for _ in range(PHILOX_ROUNDS):
            p0 = x0.astype(np.uint64) * m0
            p1 = x2.astype(np.uint64) * m1
            x0, x1, x2, x3 = ((p1 >> sh).astype(np.uint32) ^ x1 ^ k0, p1.astype(np.uint32),
                              (p0 >> sh).astype(np.uint32) ^ x3 ^ k1, p0.astype(np.uint32))
            k0 = k0 + w0
            k1 = k1 + w1
    return x0, x1, x2, x3


def to_uniform(word):
    """(w + 1) * 2**-32 on (0, 1]; rng.py:121-129."""
    if isinstance(word, np.ndarray):
        return (word.astype(np.float64) + 1.0) * TWO_NEG_32
    return (float(word) + 1.0) * TWO_NEG_32


def box_muller(u1, u2):
    """rng.py:132-142."""
    r = math.sqrt(-2.0 * math.log(u1))
    a = TWO_PI * u2
    return (r * math.cos(a), r * math.sin(a))


def gaussian_from_words(w0, w1, w2, w3, m):
    """Uniform map + Box-Muller over word blocks; rng.py:175-188.

    ``w*`` have shape (G, nblocks); returns (G, m) with the surplus of the
    last block discarded (prefix-stable in m).
    """
    u0, u1, u2, u3 = (to_uniform(np.asarray(w)) for w in (w0, w1, w2, w3))
    r_a = np.sqrt(-2.0 * np.log(u0))
    r_b = np.sqrt(-2.0 * np.log(u2))
    ang_a = TWO_PI * u1
    ang_b = TWO_PI * u3
    draws = np.stack([r_a * np.cos(ang_a), r_a * np.sin(ang_a),
                      r_b * np.cos(ang_b), r_b * np.sin(ang_b)], axis=-1)
    g = draws.shape[0]
    return draws.reshape(g, -1)[:, :m]


def normals_for_orbits(seed, orbits, chunk, step, m):
    """Per-step Philox normals; rng.py:150-188 (engine passes chunk=step>>32,
    step=step&mask, engine.py:236-240)."""
    orbits = np.asarray(orbits, dtype=np.uint32)
    if m == 0:
        return np.empty((orbits.size, 0), dtype=np.float64)
    if chunk == SAMPLING_TAG:
        raise ValueError("counter word 0x%08X is reserved for sampling streams" % SAMPLING_TAG)
    nblocks = -(-m // 4)
    seed &= MASK64
    w = philox_words(seed & MASK32, orbits[:, None], seed >> 32, chunk, step,
                     np.arange(nblocks, dtype=np.uint32)[None, :])
    return gaussian_from_words(*w, m)


def sampling_uniforms(seed, orbits, count):
    """Reserved-tag uniforms on [0, 1); rng.py:200-222."""
    orbits = np.asarray(orbits, dtype=np.uint32)
    if count == 0:
        return np.empty((orbits.size, 0), dtype=np.float64)
    nblocks = -(-count // 4)
    seed &= MASK64
    words = philox_words(seed & MASK32, orbits[:, None], seed >> 32, SAMPLING_TAG, 0,
                         np.arange(nblocks, dtype=np.uint32)[None, :])
    u = np.stack([w.astype(np.float64) * TWO_NEG_32 for w in words], axis=-1)
    return u.reshape(orbits.size, 4 * nblocks)[:, :count]


def sample_kuramoto_batch(n, orbits, omega_range, noise_range, coupling, seed, orbit_ids=None):
    """model.py:242-270; returns (init, params).  ``orbit_ids`` generalises the
    reference's arange(M) (model.py:262) to an arbitrary shard."""
    ids = np.arange(orbits, dtype=np.uint32) if orbit_ids is None else np.asarray(orbit_ids, np.uint32)
    u = sampling_uniforms(seed, ids, 3 * n)
    theta0 = -math.pi + 2.0 * math.pi * u[:, :n]
    omega = omega_range[0] + (omega_range[1] - omega_range[0]) * u[:, n:2 * n]
    strengths = noise_range[0] + (noise_range[1] - noise_range[0]) * u[:, 2 * n:]
    params = np.empty((ids.size, 2 * n + 1), dtype=np.float64)
    params[:, 0] = coupling
    params[:, 1:n + 1] = omega
    params[:, n + 1:] = strengths
    return theta0, params


# ---------------------------------------------------------------------------
# SplitMix64 / sfc64 / xoshiro256++ (not in the reference)

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)
STREAM_SALT = 0x243F6A8885A308D3


def _u64(x):
    return np.asarray(x, dtype=np.uint64)


def mix64(z):
    """SplitMix64 output finaliser (Steele, Lea & Flood 2014)."""
    z = _u64(z)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
    return z ^ (z >> np.uint64(31))


def splitmix64_outputs(x0, count):
    """First ``count`` SplitMix64 outputs from state x0: mix64(x0 + k*gamma), k=1.."""
    x0 = _u64(x0)
    out = []
    with np.errstate(over="ignore"):
        for k in range(1, count + 1):
            out.append(mix64(x0 + np.uint64(k) * _GAMMA))
    return out


def stream_origin(seed, orbit, block):
    """Per-(orbit, block) SplitMix64 origin: mix64(seed ^ mix64(id ^ salt)),
    id = orbit << 32 | block.  Depends only on the global address, so noise
    never depends on GPU count, shard boundaries or the lane layout."""
    sid = (_u64(orbit) << np.uint64(32)) | _u64(block)
    return mix64(_u64(seed & MASK64) ^ mix64(sid ^ np.uint64(STREAM_SALT)))


def rotl64(x, k):
    x = _u64(x)
    return (x << np.uint64(k)) | (x >> np.uint64(64 - k))


def sfc64_next(s):
    """numpy's sfc64_next: s = [a, b, c, counter] (uint64 arrays, updated in place)."""
    a, b, c, w = s
    with np.errstate(over="ignore"):
        tmp = a + b + w
        s[3] = w + np.uint64(1)
        s[0] = b ^ (b >> np.uint64(11))
        s[1] = c + (c << np.uint64(3))
        s[2] = rotl64(c, 24) + tmp
    return tmp


def sfc64_seed_words(a, b, c):
    """numpy's sfc64_set_seed: (a, b, c, counter=1) then 12 discarded outputs."""
    s = [_u64(a).copy(), _u64(b).copy(), _u64(c).copy(), np.ones_like(_u64(a))]
    for _ in range(12):
        sfc64_next(s)
    return s


def xoshiro256pp_next(s):
    """xoshiro256++ (Blackman & Vigna 2019); s = [s0, s1, s2, s3] updated in place."""
    s0, s1, s2, s3 = s
    with np.errstate(over="ignore"):
        result = rotl64(s0 + s3, 23) + s0
    t = s1 << np.uint64(17)
    s2 = s2 ^ s0
    s3 = s3 ^ s1
    s1 = s1 ^ s2
    s0 = s0 ^ s3
    s2 = s2 ^ t
    s3 = rotl64(s3, 45)
    s[0], s[1], s[2], s[3] = s0, s1, s2, s3
    return result


def stream_init(stream, seed, orbit, block):
    """Initial 4x uint64 state of stream (orbit, block); arrays broadcast."""
    o = splitmix64_outputs(stream_origin(seed, orbit, block), 4)
    if stream == "sfc64":
        return sfc64_seed_words(o[0], o[1], o[2])
    if stream == "xoshiro256pp":
        return [o[0], o[1], o[2], o[3]]
    raise ValueError("stateful stream expected, got %r" % (stream,))


def stream_next(stream, s):
    return sfc64_next(s) if stream == "sfc64" else xoshiro256pp_next(s)


def stream_block_words(stream, s):
    """One 4-word block: two 64-bit outputs split (lo32, hi32)."""
    o1 = stream_next(stream, s)
    o2 = stream_next(stream, s)
    m = np.uint64(MASK32)
    sh = np.uint64(32)
    return ((o1 & m).astype(np.uint32), (o1 >> sh).astype(np.uint32),
            (o2 & m).astype(np.uint32), (o2 >> sh).astype(np.uint32))


def stream_raw(stream, seed, orbit, block, count):
    """First ``count`` raw 64-bit outputs of one stream."""
    s = stream_init(stream, seed, np.array([orbit], np.uint64), np.array([block], np.uint64))
    return np.array([int(stream_next(stream, s)[0]) for _ in range(count)], dtype=np.uint64)


# ---------------------------------------------------------------------------
# Kuramoto model (model.py:188-201) and steppers (solvers.py:63-88)

def kuramoto_drift(y, p):
    """model.py:188-196, same op order (pairwise numpy sum over the row)."""
    n = y.shape[-1]
    pairwise = np.subtract(y[..., None, :], y[..., :, None])
    np.sin(pairwise, out=pairwise)
    coupling = np.sum(pairwise, axis=-1)
    return np.add(p[..., 1:n + 1], np.multiply(np.divide(p[..., 0:1], float(n)), coupling))


def kuramoto_diffusion(y, p, noise):
    """model.py:199-201."""
    n = y.shape[-1]
    return np.multiply(p[..., n + 1:2 * n + 1], noise)


def em_step(y, p, dt, noise):
    """solvers.py:63-71: (y + f*dt) + sqrt(dt)*g."""
    return y + kuramoto_drift(y, p) * dt + np.sqrt(dt) * kuramoto_diffusion(y, p, noise)


def euler_step(y, p, dt):
    """solvers.py:74-77."""
    return y + kuramoto_drift(y, p) * dt


def rk4_step(y, p, dt):
    """solvers.py:80-88."""
    half = 0.5 * dt
    k1 = kuramoto_drift(y, p)
    k2 = kuramoto_drift(y + half * k1, p)
    k3 = kuramoto_drift(y + half * k2, p)
    k4 = kuramoto_drift(y + dt * k3, p)
    return y + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)


def iteration_count(tspan, dt, ksteps, pad=False):
    """engine.py:126-142."""
    ratio = tspan / (dt * ksteps)
    k = round(ratio)
    if k >= 1 and abs(ratio - k) <= 1e-9 * max(1.0, abs(ratio)):
        return k
    if pad:
        return max(1, math.ceil(ratio - 1e-12))
    raise ValueError("tspan is not an integer multiple of dt*ksteps")


# ---------------------------------------------------------------------------
# The restated run loop (engine.py:184-277)

def integrate(init, params, *, dt, ksteps, chunks, seed=0, solver="em", nnoise=None,
              stream="philox", orbit_ids=None, threads=1, group=None, drift=None,
              diffusion=None):
    """Restated ``run_batch`` inner loop for global ``orbit_ids``.

    engine.py:223-263 (integrate_group) with the stepper of engine.py:153-181.
    Returns (times, values, failures) where failures are
    (orbit, chunk, step, time, reason) tuples sorted by orbit (engine.py:275).
    ``threads``/``group`` mirror the reference's pool over contiguous orbit
    groups (engine.py:265-274); they never change the result.  ``drift(t, y,
    p)`` / ``diffusion(t, y, p, noise)`` default to the Kuramoto system; pass
    :func:`expression_model` functions for a template model.
    """
    f_drift = drift if drift is not None else (lambda t, y, p: kuramoto_drift(y, p))
    f_diff = diffusion if diffusion is not None else (
        lambda t, y, p, noise: kuramoto_diffusion(y, p, noise))
    init = np.asarray(init, dtype=np.float64)
    params = np.asarray(params, dtype=np.float64)
    m_orbits, n = init.shape
    if nnoise is None:
        nnoise = n if solver == "em" else 0
    ids = (np.arange(m_orbits, dtype=np.uint64) if orbit_ids is None
           else np.asarray(orbit_ids, dtype=np.uint64))
    samples = chunks + 1
    times = np.arange(samples, dtype=np.float64) * (ksteps * dt)
    values = np.empty((m_orbits, samples, n), dtype=np.float64)
    values[:, 0, :] = init
    stochastic = solver == "em" and nnoise > 0
    nblocks = -(-nnoise // 4) if nnoise else 0
    sqrt_dt = np.sqrt(dt)

    def run_group(lo, hi):
        y = init[lo:hi].copy()
        p = params[lo:hi]
        gids = ids[lo:hi]
        alive = np.ones(hi - lo, dtype=bool)
        fails = []
        st = None
        if stochastic and stream != "philox":
            st = stream_init(stream, seed, gids[:, None],
                             np.arange(nblocks, dtype=np.uint64)[None, :])
        with np.errstate(all="ignore"):
            for chunk in range(chunks):
                for local in range(ksteps):
                    s = chunk * ksteps + local
                    t = s * dt
                    if stochastic:
                        if st is None:
                            noise = normals_for_orbits(seed, gids.astype(np.uint32),
                                                       (s >> 32) & MASK32, s & MASK32, nnoise)
                        else:
                            noise = gaussian_from_words(*stream_block_words(stream, st), nnoise)
                        y = (y + f_drift(t, y, p) * dt) + sqrt_dt * f_diff(t, y, p, noise)
                    elif solver in ("em", "euler"):
                        y = y + f_drift(t, y, p) * dt
                    elif solver == "rk4":
                        half = 0.5 * dt
                        k1 = f_drift(t, y, p)
                        k2 = f_drift(t + half, y + half * k1, p)
                        k3 = f_drift(t + half, y + half * k2, p)
                        k4 = f_drift(t + dt, y + dt * k3, p)
                        y = y + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
                    else:
                        raise ValueError("unsupported solver %r" % (solver,))
                    ok = np.isfinite(y).all(axis=-1)
                    failed = alive & ~ok
                    if failed.any():
                        for idx in np.nonzero(failed)[0]:
                            fails.append((int(gids[idx]), chunk, local, t,
                                          "state became non-finite"))
                        y[failed] = np.nan
                        alive = alive & ok
                values[lo:hi, chunk + 1, :] = y
        return fails

    group = m_orbits if group is None else group
    bounds = [(lo, min(lo + group, m_orbits)) for lo in range(0, m_orbits, group)]
    failures = []
    if threads <= 1 or len(bounds) == 1:
        for lo, hi in bounds:
            failures.extend(run_group(lo, hi))
    else:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            for res in pool.map(lambda b: run_group(*b), bounds):
                failures.extend(res)
    failures.sort(key=lambda f: f[0])
    return times, values, failures


# ---------------------------------------------------------------------------
# Expression templates (dsl.py:1-27 grammar; interpreter dsl.py:441-571)
#
# Parsing goes through Python's own expression parser: with '^' spelled '**'
# the template grammar is a subset of Python's with the same precedences
# (unary minus looser than '**', '**' right-associative and taking a signed
# right operand).  Evaluation restates the reference interpreter: numpy
# float64 ufuncs, equation index i and sum indices as int64 arrays on their
# own broadcast axes, indexing through np.take, sums as np.sum over the last
# axis (numpy pairwise order).

_EXPR_FUNCS = {"sin": np.sin, "cos": np.cos, "tan": np.tan, "exp": np.exp, "ln": np.log,
               "sqrt": np.sqrt, "abs": np.abs}
_EXPR_BIN = {"Add": np.add, "Sub": np.subtract, "Mult": np.multiply, "Div": np.divide,
             "Pow": np.power}


def _expr_tree(text):
    import ast
    return ast.parse(text.replace("^", "**"), mode="eval").body


def _expr_index(node, axes):
    """dsl.py:472-496: integer index arithmetic."""
    import ast
    if isinstance(node, ast.Constant):
        return int(node.value)
    if isinstance(node, ast.Name):
        if node.id == "N":
            return axes["N"]
        return axes[node.id]
    if isinstance(node, ast.UnaryOp):
        return -_expr_index(node.operand, axes)
    a, b = _expr_index(node.left, axes), _expr_index(node.right, axes)
    op = type(node.op).__name__
    return a + b if op == "Add" else a - b if op == "Sub" else a * b


def _expr_eval(node, env, axes, depth):
    """dsl.py:441-551 (_Evaluator.eval) for one expression node."""
    import ast
    if isinstance(node, ast.Constant):
        return float(node.value)
    if isinstance(node, ast.Name):
        if node.id == "t":
            return env["t"]
        if node.id == "N":
            return float(env["N"])
        return axes[node.id]
    if isinstance(node, ast.UnaryOp):
        return np.negative(_expr_eval(node.operand, env, axes, depth))
    if isinstance(node, ast.BinOp):
        left = _expr_eval(node.left, env, axes, depth)
        right = _expr_eval(node.right, env, axes, depth)
        return _EXPR_BIN[type(node.op).__name__](left, right)
    if isinstance(node, ast.Subscript):
        arr = env[node.value.id]
        idx = _expr_index(node.slice, axes)
        taken = np.take(arr, idx, axis=-1)
        if not isinstance(idx, np.ndarray) and depth:
            taken = np.reshape(taken, np.shape(taken) + (1,) * depth)
        return taken
    if isinstance(node, ast.Call):
        name = node.func.id
        if name == "sum":  # dsl.py:533-551
            var = node.args[0].id
            n = env["N"]
            inner = {k: (v.reshape(v.shape + (1,)) if isinstance(v, np.ndarray) else v)
                     for k, v in axes.items()}
            inner[var] = np.arange(n, dtype=np.int64).reshape((1,) * depth + (n,))
            body = np.asarray(_expr_eval(node.args[1], env, inner, depth + 1))
            full = np.broadcast_shapes(body.shape, (1,) * depth + (n,))
            if body.shape != full:
                body = np.broadcast_to(body, full)
            return np.sum(body, axis=-1)
        return _EXPR_FUNCS[name](_expr_eval(node.args[0], env, axes, depth))
    raise ValueError("unsupported expression node %r" % (node,))


def evaluate_expression(text, t, y, p, noise=None):
    """All equations of a template at once (dsl.evaluate with i=None)."""
    y = np.asarray(y, dtype=np.float64)
    n = y.shape[-1]
    env = {"t": float(t), "N": n, "y": y, "p": np.asarray(p, dtype=np.float64), "n": noise}
    axes = {"i": np.arange(n, dtype=np.int64), "N": n}
    with np.errstate(all="ignore"):
        out = _expr_eval(_expr_tree(text), env, axes, 1)
    return np.broadcast_to(np.asarray(out, dtype=np.float64), y.shape)


def expression_model(drift_text, diffusion_text=None):
    """(drift, diffusion) callables for :func:`integrate` from template text
    (model.py:142-182: results broadcast to the state's shape)."""
    def drift(t, y, p):
        return evaluate_expression(drift_text, t, y, p)

    def diffusion(t, y, p, noise):
        return evaluate_expression(diffusion_text, t, y, p, noise)
    return drift, diffusion


# ---------------------------------------------------------------------------
# Analysis (analysis.py:72-186)

def wrap_phase(x):
    """analysis.py:72-74: onto [-pi, pi)."""
    return np.mod(np.asarray(x, dtype=np.float64) + math.pi, 2.0 * math.pi) - math.pi


def order_parameter_arrays(phases):
    """analysis.py:77-82: r = min(|mean(e^{i theta})|, 1), Phi wrapped, Phi = 0 at r = 0."""
    z = np.exp(1j * np.asarray(phases, dtype=np.float64)).mean(axis=-1)
    r = np.minimum(np.abs(z), 1.0)
    phi = wrap_phase(np.arctan2(z.imag, z.real))
    return r, np.where(r == 0.0, 0.0, phi)


def ensemble_mean_std(r):
    """analysis.py:126-130: per-time mean and population std over realizations."""
    r = np.asarray(r, dtype=np.float64)
    return r.mean(axis=0), r.std(axis=0)


def mixed_error(got, ref):
    """max |got - ref| / max(1, |ref|) -- the parity metric (north_star 1e-10).
    NaNs must coincide; returns inf otherwise."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if got.shape != ref.shape:
        return math.inf
    gn, rn = np.isnan(got), np.isnan(ref)
    if not np.array_equal(gn, rn):
        return math.inf
    gi, ri = np.isinf(got), np.isinf(ref)
    if not np.array_equal(gi, ri) or not np.array_equal(got[ri], ref[ri]):
        return math.inf
    mask = ~(rn | ri)
    if not mask.any():
        return 0.0
    d = np.abs(got[mask] - ref[mask]) / np.maximum(1.0, np.abs(ref[mask]))
    return float(d.max())
