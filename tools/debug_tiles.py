"""Diagnose host-pipeline tiling differences (rows / samples that differ)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1908_03869_b200 as sdb  # noqa: E402
from paper_1908_03869_b200 import EngineConfig, OrbitBatch, run_batch  # noqa: E402
from paper_1908_03869_b200.engine import last_launch_info  # noqa: E402

n, m = 16, 1501
batch = sdb.sample_kuramoto_batch(n, m, (0.2, 0.4), (0.01, 0.1), 0.3, seed=11)
params = batch.params.copy()
params[1000, 1 + 5] = 1e308
batch = OrbitBatch(init=batch.init, params=params)
for stream in ("philox", "sfc64"):
    cfg = EngineConfig(dt=1e-2, tspan=2.0, ksteps=20, orbits=m, seed=2, stream=stream)
    ref = run_batch(sdb.kuramoto_model(n), cfg, batch)
    print(stream, "ref", last_launch_info())
    ref2 = run_batch(sdb.kuramoto_model(n), cfg, batch)
    print(" ref repeat same:", np.array_equal(ref.values, ref2.values, equal_nan=True))
    for tiles, piece_kb, threads in [(1, 65536, 1), (3, 65536, 1), (3, 100, 4), (7, 40, 1), (2, 65536, 8), (1, 1, 2)]:
        os.environ["SDEB200_TILES"] = str(tiles)
        os.environ["SDEB200_PIECE_KB"] = str(piece_kb)
        os.environ["SDEB200_HOST_THREADS"] = str(threads)
        got = run_batch(sdb.kuramoto_model(n), cfg, batch)
        info = last_launch_info()
        diff = ~((got.values == ref.values) | (np.isnan(got.values) & np.isnan(ref.values)))
        rows = np.nonzero(diff.any(axis=(1, 2)))[0]
        samp = np.nonzero(diff.any(axis=(0, 2)))[0]
        print(" tiles=%d piece=%dKB thr=%d info=%s: %d rows differ %s samples %s maxabs %.3g fails %s/%s" % (
            tiles, piece_kb, threads, info, len(rows), rows[:10], samp[:12],
            np.nanmax(np.abs(got.values - ref.values)) if len(rows) else 0.0,
            [f.orbit for f in got.failures], [f.orbit for f in ref.failures]))
    for k in ("SDEB200_TILES", "SDEB200_PIECE_KB", "SDEB200_HOST_THREADS"):
        del os.environ[k]
