"""sdeb200 -- B200-native ensemble SDE integrator (drop-in for ``sdebatch``).

The public names on the reference's hot path (/root/reference/pkg/src/
sdebatch/__init__.py:11-22) with the same signatures; integration, noise
generation and batch sampling run as hand-written sm_100a CUDA kernels in
libsdeb200.so (C ABI: include/sdeb200.h).  There is no CPU fallback.
"""

__version__ = "0.1.0"

from .model import (ModelSpec, OrbitBatch, ModelDefinitionError, kuramoto_model,
                    kuramoto_dsl_model, sample_kuramoto_batch, speed_protocol_batch,
                    accuracy_protocol_batch, model_from_name, model_from_file,
                    model_from_dsl, drift_eval, diffusion_eval, pin_batch)
from .engine import (EngineConfig, TrajectoryStore, OrbitFailure, ConfigError, run_batch,
                     iteration_count, partition_orbits)
from .solvers import (euler_maruyama_step, euler_step, rk4_step, implicit_euler_step,
                      implicit_midpoint_step, get_solver, SOLVERS)
from .storage import store_hash, write_store, read_store, run_batch_to_file
from .analysis import (CoherencePoint, CoherenceSeries, EnsembleStats, order_parameter,
                       coherence_series, ensemble_stats, dt_sweep, kymograph_export, wrap_phase,
                       run_coherence)
from . import analysis, dsl, rng, storage

__all__ = [
    "__version__",
    "ModelSpec", "OrbitBatch", "ModelDefinitionError", "kuramoto_model", "kuramoto_dsl_model",
    "sample_kuramoto_batch", "speed_protocol_batch", "accuracy_protocol_batch",
    "model_from_name", "model_from_file", "model_from_dsl", "drift_eval", "diffusion_eval",
    "pin_batch",
    "EngineConfig", "TrajectoryStore", "OrbitFailure", "ConfigError", "run_batch",
    "iteration_count", "partition_orbits",
    "euler_maruyama_step", "euler_step", "rk4_step",
    "implicit_euler_step", "implicit_midpoint_step", "get_solver", "SOLVERS",
    "store_hash", "write_store", "read_store", "run_batch_to_file", "storage",
    "dsl", "rng", "analysis",
    "CoherencePoint", "CoherenceSeries", "EnsembleStats", "order_parameter", "coherence_series",
    "ensemble_stats", "dt_sweep", "kymograph_export", "wrap_phase", "run_coherence",
]
