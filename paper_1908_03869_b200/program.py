"""Compiled expression-template models: the device side of ``model_from_dsl``.

A model whose drift/diffusion are expression templates (model.py:291-309) is
handed to libsdeb200 as canonical template text (``dsl.to_source``); the
library generates CUDA device functions and builds them with NVRTC for
sm_100a (``sdb_model_*`` in include/sdeb200.h).  This module keeps one
compiled handle per (dimensions, drift, diffusion), and performs the checks
the reference makes while interpreting (dsl.py:489-531): every index an
expression can take over the evaluated equation range must be in bounds, else
:class:`dsl.DomainError` -- the device does not bounds-check.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native as nat
from . import dsl

_models: dict = {}
_models_lock = threading.Lock()

WHICH_DRIFT, WHICH_DIFFUSION = 0, 1


class CompiledModel:
    """An sdb_model handle (freed with the object)."""

    def __init__(self, nequat: int, nparams: int, nnoise: int, drift: str, diffusion: str):
        self.nequat, self.nparams, self.nnoise = nequat, nparams, nnoise
        self.drift, self.diffusion = drift, diffusion
        handle = ctypes.c_void_p()
        nat.check(nat.lib().sdb_model_create(nequat, nparams, nnoise, drift.encode(),
                                             diffusion.encode(), ctypes.byref(handle)),
                  None, "sdb_model_create")
        self.handle = handle.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and nat is not None and nat._lib is not None:
            nat.lib().sdb_model_free(h)
            self.handle = None

    def source(self, kind: int, factored: bool = False) -> str:
        """Generated CUDA of one program kind (factored: the meanfield form
        run_batch uses with coupling="meanfield")."""
        k = kind | (256 if factored else 0)
        n = nat.lib().sdb_model_source(self.handle, k, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        nat.lib().sdb_model_source(self.handle, k, buf, n + 1)
        return buf.value.decode()

    def build(self, kind: int, factored: bool = False):
        """NVRTC-compile one program kind (no GPU needed)."""
        nat.check(nat.lib().sdb_model_build(self.handle, kind | (256 if factored else 0)), None,
                  "sdb_model_build")


def compiled(nequat: int, nparams: int, nnoise: int, drift, diffusion) -> CompiledModel:
    """Cached compiled model for template ASTs/text (diffusion None -> "0")."""
    dtext = dsl.to_source(dsl.as_ast(drift))
    gtext = "0.0" if diffusion is None else dsl.to_source(dsl.as_ast(diffusion))
    key = (int(nequat), int(nparams), int(nnoise), dtext, gtext)
    with _models_lock:
        m = _models.get(key)
        if m is None:
            m = CompiledModel(*key)
            _models[key] = m
        return m


def model_program(model) -> CompiledModel:
    return compiled(model.nequat, model.nparams, model.nnoise, model.drift,
                    model.diffusion if model.nnoise > 0 else None)


# ---------------------------------------------------------------------------
# index bounds (the reference checks them while evaluating, dsl.py:489-531)

def _index_values(node, env):
    """Integer value(s) of an index sub-expression over the bound variables
    (numpy int64 arrays on separate broadcast axes)."""
    if isinstance(node, dsl.Num):
        if not float(node.value).is_integer():
            raise dsl.DomainError("non-integer constant in index expression", node.pos)
        return np.int64(int(node.value))
    if isinstance(node, dsl.Var):
        if node.name in env:
            return env[node.name]
        raise dsl.DomainError("unknown variable %r in index expression" % node.name, node.pos)
    if isinstance(node, dsl.Neg):
        return -_index_values(node.operand, env)
    if isinstance(node, dsl.BinOp) and node.op in "+-*":
        a, b = _index_values(node.left, env), _index_values(node.right, env)
        return a + b if node.op == "+" else a - b if node.op == "-" else a * b
    raise dsl.DomainError("index expressions must be integer arithmetic", node.pos)


def check_indices(expr, n: int, dims: dict, equations) -> None:
    """Raise DomainError if any y/p/n index of ``expr`` leaves its vector for
    an equation index in ``equations`` and every enclosing sum index."""
    depth = [0]

    def walk(node, env):
        if isinstance(node, dsl.Index):
            length = dims.get(node.base)
            if length is None:
                raise dsl.DomainError("noise vector is not available in this context", node.pos)
            idx = np.asarray(_index_values(node.index, env))
            if idx.size and (idx.min() < 0 or idx.max() >= length):
                raise dsl.DomainError("index out of range for %s (length %d)"
                                      % (node.base, length), node.pos)
            walk(node.index, env)
        elif isinstance(node, dsl.Sum):
            depth[0] += 1
            shape = (1,) * depth[0] + (n,)
            inner = {k: (v.reshape(v.shape + (1,)) if isinstance(v, np.ndarray) else v)
                     for k, v in env.items()}
            inner[node.var] = np.arange(n, dtype=np.int64).reshape(shape)
            walk(node.body, inner)
            depth[0] -= 1
        elif isinstance(node, dsl.Neg):
            walk(node.operand, env)
        elif isinstance(node, dsl.BinOp):
            walk(node.left, env)
            walk(node.right, env)
        elif isinstance(node, dsl.Call):
            walk(node.arg, env)

    walk(dsl.as_ast(expr), {"i": np.asarray(list(equations), dtype=np.int64), "N": np.int64(n)})


def check_model_indices(model) -> None:
    """run_batch's pre-flight for template models: every equation's indices
    in range (the reference raises the same DomainError at the first step)."""
    n = model.nequat
    eqs = range(n)
    check_indices(model.drift, n, {"y": n, "p": model.nparams}, eqs)
    if model.nnoise > 0:
        check_indices(model.diffusion, n, {"y": n, "p": model.nparams, "n": model.nnoise}, eqs)


# ---------------------------------------------------------------------------
# device entry points

def _flat(a, lead, width):
    return nat.f64(np.broadcast_to(a, lead + (width,)).reshape(-1, width))


def eval_rows(cm: CompiledModel, which: int, t: float, y, p, noise=None):
    """drift (which=0) / diffusion (1) on the device over broadcast rows."""
    y = np.asarray(y, dtype=np.float64)
    p = np.asarray(p, dtype=np.float64)
    shapes = [y.shape[:-1], p.shape[:-1]]
    if noise is not None:
        noise = np.asarray(noise, dtype=np.float64)
        shapes.append(noise.shape[:-1])
    lead = np.broadcast_shapes(*shapes)
    yy = _flat(y, lead, cm.nequat)
    pp = _flat(p, lead, cm.nparams) if cm.nparams else np.zeros((yy.shape[0], 1))
    nz = _flat(noise, lead, cm.nnoise) if (noise is not None and cm.nnoise) else None
    out = np.empty_like(yy)
    ctx = nat.context()
    nat.check(nat.lib().sdb_model_eval(ctx, cm.handle, which, float(t), yy.shape[0], nat.dptr(yy),
                                       nat.dptr(pp), nat.dptr(nz) if nz is not None else None,
                                       nat.dptr(out)), ctx, "sdb_model_eval")
    return out.reshape(lead + (cm.nequat,))


def step_rows(cm: CompiledModel, solver: str, t: float, y, p, dt: float, noise=None):
    y = np.asarray(y, dtype=np.float64)
    p = np.asarray(p, dtype=np.float64)
    shapes = [y.shape[:-1], p.shape[:-1]]
    if noise is not None:
        noise = np.asarray(noise, dtype=np.float64)
        shapes.append(noise.shape[:-1])
    lead = np.broadcast_shapes(*shapes)
    yy = _flat(y, lead, cm.nequat)
    pp = _flat(p, lead, cm.nparams) if cm.nparams else np.zeros((yy.shape[0], 1))
    nz = _flat(noise, lead, cm.nnoise) if (noise is not None and cm.nnoise) else None
    out = np.empty_like(yy)
    ctx = nat.context()
    nat.check(nat.lib().sdb_model_step(ctx, cm.handle, nat.SOLVER_IDS[solver], float(t),
                                       float(dt), yy.shape[0], nat.dptr(yy), nat.dptr(pp),
                                       nat.dptr(nz) if nz is not None else None, nat.dptr(out)),
              ctx, "sdb_model_step")
    return out.reshape(lead + (cm.nequat,))


def _bind_i(node, value: int):
    if isinstance(node, dsl.Var):
        return dsl.Num(float(value), node.pos) if node.name == "i" else node
    if isinstance(node, dsl.Index):
        return dsl.Index(node.base, _bind_i(node.index, value), node.pos)
    if isinstance(node, dsl.Neg):
        return dsl.Neg(_bind_i(node.operand, value), node.pos)
    if isinstance(node, dsl.BinOp):
        return dsl.BinOp(node.op, _bind_i(node.left, value), _bind_i(node.right, value), node.pos)
    if isinstance(node, dsl.Call):
        return dsl.Call(node.func, _bind_i(node.arg, value), node.pos)
    if isinstance(node, dsl.Sum):
        return dsl.Sum(node.var, _bind_i(node.body, value), node.pos)
    return node


def evaluate_expression(expr, ctx, strict: bool):
    """dsl.evaluate on the device: the expression becomes the drift (or, with
    a noise vector, the diffusion) of a one-off compiled model."""
    n = int(ctx.N)
    y = np.asarray(ctx.y, dtype=np.float64)
    p = np.asarray(ctx.p, dtype=np.float64)
    noise = None if ctx.n is None else np.asarray(ctx.n, dtype=np.float64)
    if ctx.i is not None and not 0 <= int(ctx.i) < n:
        raise ValueError("equation index i=%r out of range for N=%r" % (ctx.i, ctx.N))
    equations = range(n) if ctx.i is None else [int(ctx.i)]
    dims = {"y": y.shape[-1], "p": p.shape[-1]}
    if noise is not None:
        dims["n"] = noise.shape[-1]
    check_indices(expr, n, dims, equations)
    text = dsl.to_source(expr)
    if ctx.i is not None:
        # one equation: bind i as a constant so every equation the program
        # evaluates is the requested one (no other i can index out of range)
        expr = _bind_i(expr, int(ctx.i))
    ny, npar = y.shape[-1], p.shape[-1]
    if ny != n:
        # evaluate on an N-wide state: pad/crop y so the program's vector has N
        # entries (indices were checked against the real length above)
        width = max(ny, n)
        yw = np.zeros(y.shape[:-1] + (width,))
        yw[..., :ny] = y
        y = yw
        if width != n:
            raise NotImplementedError("evaluate with y longer than N is not supported on the "
                                      "device path")
    if noise is not None:
        cm = compiled(n, npar, noise.shape[-1], "0.0", expr)
        out = eval_rows(cm, WHICH_DIFFUSION, ctx.t, y, p, noise)
    else:
        cm = compiled(n, npar, 0, expr, None)
        out = eval_rows(cm, WHICH_DRIFT, ctx.t, y, p)
    if strict:
        inputs = [y, p] + ([noise] if noise is not None else [])
        finite_in = all(np.isfinite(a).all() for a in inputs) and np.isfinite(ctx.t)
        sel = out if ctx.i is None else out[..., int(ctx.i)]
        if finite_in and not np.isfinite(sel).all():
            raise dsl.DomainError("domain error in %r (non-finite result)" % text,
                                  getattr(expr, "pos", (0, 0)))
    if ctx.i is None:
        return out
    res = out[..., int(ctx.i)]
    return float(res) if np.ndim(res) == 0 else res
