import ctypes
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
ORACLE_STREAMS_LIB = os.path.join(ROOT, "oracle", "_build", "liboracle_streams.so")

# the parity bar of north_star: |got - ref| <= 1e-10 * max(1, |ref|) in FP64
PARITY_TOL = 1e-10


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsdeb200.so")
    # the layout autotuner's on-disk cache: a per-session file, so every test
    # session probes like a fresh box and nothing lands in ~/.cache
    if "SDEB200_TUNE_CACHE" not in os.environ:
        import tempfile
        os.environ["SDEB200_TUNE_CACHE"] = os.path.join(
            tempfile.mkdtemp(prefix="sdeb200-tune-"), "layouts.tsv")


@pytest.fixture(scope="session")
def golden():
    data = np.load(os.path.join(GOLDEN_DIR, "golden_v1.npz"))
    with open(os.path.join(GOLDEN_DIR, "cases.json")) as fh:
        cases = json.load(fh)
    return {k: data[k] for k in data.files}, cases


@pytest.fixture(scope="session")
def cstreams():
    """The C restatement of the noise generators (oracle/streams.c)."""
    if not os.path.exists(ORACLE_STREAMS_LIB):
        import subprocess
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True,
                       capture_output=True)
    lib = ctypes.CDLL(ORACLE_STREAMS_LIB)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    u32p = ctypes.POINTER(ctypes.c_uint32)
    lib.oracle_stream_raw.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_int64, u64p]
    lib.oracle_stream_raw_from_state.argtypes = [ctypes.c_int, u64p, ctypes.c_int64, u64p]
    lib.oracle_sfc64_set_seed.argtypes = [u64p, u64p]
    lib.oracle_philox.argtypes = [u32p, u32p, u32p]
    return lib


def case_config(case):
    """EngineConfig kwargs of a golden case (seed stored as a string)."""
    cfg = dict(case["config"])
    cfg["seed"] = int(cfg["seed"])
    return cfg


@pytest.fixture(scope="session")
def golden_dsl():
    """Reference run_batch / drift_eval outputs for expression-template models
    (tests/golden/make_golden_dsl.py)."""
    data = np.load(os.path.join(GOLDEN_DIR, "golden_dsl_v1.npz"))
    with open(os.path.join(GOLDEN_DIR, "cases_dsl.json")) as fh:
        cases = json.load(fh)
    return {k: data[k] for k in data.files}, cases


@pytest.fixture(scope="session")
def golden_analysis():
    """Reference analysis outputs (tests/golden/make_golden_analysis.py)."""
    data = np.load(os.path.join(GOLDEN_DIR, "golden_analysis_v1.npz"))
    with open(os.path.join(GOLDEN_DIR, "cases_analysis.json")) as fh:
        cases = json.load(fh)
    return {k: data[k] for k in data.files}, cases
