"""Single-step integrators (drop-in for ``sdebatch.solvers``,
/root/reference/pkg/src/sdebatch/solvers.py).

em / euler / rk4 run on the GPU with the reference's operation order
(solvers.py:63-88): sdb_step for the Kuramoto system, the compiled program's
step kernel (sdb_model_step) for expression-template models.  The implicit fixed-point steppers (ie, im;
solvers.py:91-137) are registered with the same metadata so configuration
validation behaves identically, but they are outside the device path this
round and raise NotImplementedError when executed.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat

__all__ = [
    "StepResult", "ConvergenceError", "SolverInfo", "SOLVERS", "get_solver",
    "euler_maruyama_step", "euler_step", "rk4_step",
    "implicit_euler_step", "implicit_midpoint_step",
]

DEFAULT_TOL = 1e-10
DEFAULT_MAX_ITER = 50


class ConvergenceError(RuntimeError):
    """solvers.py:45-51."""

    def __init__(self, message: str, t: float, iterations: int):
        super().__init__(message)
        self.t = t
        self.iterations = iterations


@dataclass(frozen=True)
class StepResult:
    y: np.ndarray
    iterations: int
    converged: np.ndarray


@dataclass(frozen=True)
class SolverInfo:
    name: str
    stochastic: bool
    implicit: bool


# solvers.py:140-161
SOLVERS = {
    "em": SolverInfo("em", stochastic=True, implicit=False),
    "euler": SolverInfo("euler", stochastic=False, implicit=False),
    "rk4": SolverInfo("rk4", stochastic=False, implicit=False),
    "ie": SolverInfo("ie", stochastic=False, implicit=True),
    "im": SolverInfo("im", stochastic=False, implicit=True),
}


def get_solver(name: str) -> SolverInfo:
    try:
        return SOLVERS[name]
    except KeyError:
        raise ValueError("unknown solver %r (choose from %s)"
                         % (name, ", ".join(sorted(SOLVERS))))


def _device_step(solver: str, model, y, p, dt, noise=None, coupling="meanfield", t=0.0):
    from .model import _check_dims, _rows, expression_model, require_kuramoto
    y = np.asarray(y, dtype=np.float64)
    p = np.asarray(p, dtype=np.float64)
    _check_dims(model, y, p)
    if expression_model(model):
        from . import program
        program.check_model_indices(model)
        if solver == "em" and model.nnoise > 0:
            noise = np.asarray(noise, dtype=np.float64)
            if noise.shape[-1] != model.nnoise:
                raise ValueError("noise vector has length %d, model has nnoise=%d"
                                 % (noise.shape[-1], model.nnoise))
        else:
            noise = None
        return program.step_rows(program.model_program(model), solver, t, y, p, dt, noise)
    n, nnoise = require_kuramoto(model)
    lead, yy, pp = _rows(y, p)
    nz = None
    if solver == "em" and nnoise > 0:
        noise = np.asarray(noise, dtype=np.float64)
        if noise.shape[-1] != nnoise:
            raise ValueError("noise vector has length %d, model has nnoise=%d"
                             % (noise.shape[-1], nnoise))
        nz = nat.f64(np.broadcast_to(noise, lead + (nnoise,)).reshape(-1, nnoise))
    out = np.empty_like(yy)
    ctx = nat.context()
    nat.check(nat.lib().sdb_step(ctx, nat.SOLVER_IDS[solver], n, model.nparams,
                                 nnoise if solver == "em" else 0, nat.COUPLING_IDS[coupling],
                                 yy.shape[0], float(dt), nat.dptr(yy), nat.dptr(pp),
                                 nat.dptr(nz) if nz is not None else None, nat.dptr(out)),
              ctx, "sdb_step")
    return out.reshape(lead + (n,))


def euler_maruyama_step(model, t: float, y, p, dt: float, noise, coupling="meanfield"):
    """One Euler-Maruyama step (solvers.py:63-71); nnoise = 0 is exactly euler."""
    if model.nnoise == 0:
        return euler_step(model, t, y, p, dt, coupling=coupling)
    return _device_step("em", model, y, p, dt, noise, coupling, t)


def euler_step(model, t: float, y, p, dt: float, coupling="meanfield"):
    """One explicit Euler step (solvers.py:74-77)."""
    return _device_step("euler", model, y, p, dt, None, coupling, t)


def rk4_step(model, t: float, y, p, dt: float, coupling="meanfield"):
    """One classical RK4 step (solvers.py:80-88)."""
    return _device_step("rk4", model, y, p, dt, None, coupling, t)


def implicit_euler_step(model, t, y, p, dt, tol=DEFAULT_TOL, max_iter=DEFAULT_MAX_ITER,
                        raise_on_failure=True):
    if tol <= 0:
        raise ValueError("tol must be positive")
    raise NotImplementedError("implicit steppers are outside the B200 device path")


def implicit_midpoint_step(model, t, y, p, dt, tol=DEFAULT_TOL, max_iter=DEFAULT_MAX_ITER,
                           raise_on_failure=True):
    if tol <= 0:
        raise ValueError("tol must be positive")
    raise NotImplementedError("implicit steppers are outside the B200 device path")
