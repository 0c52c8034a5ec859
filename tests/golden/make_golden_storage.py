"""Golden store files written by the REFERENCE's storage module (build
container only): CSV and SDB1 files of a seeded store, compared byte for byte
with this package's writers (tests/test_storage_host.py).

    python tests/golden/make_golden_storage.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("SDEBATCH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from sdebatch import storage  # noqa: E402
from sdebatch.engine import TrajectoryStore  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
g = np.random.default_rng(99)
values = g.standard_normal((3, 4, 2)) * np.array([1.0, 1e-7])
values[1, 2, 0] = np.nan
values[2, 3, 1] = 1e300
times = np.arange(4, dtype=np.float64) * 0.25
store = TrajectoryStore(times=times, values=values, model_name="golden-store")
storage.write_store(store, os.path.join(HERE, "store_ref.csv"), fmt="csv")
storage.write_store(store, os.path.join(HERE, "store_ref.sdb1"), fmt="bin",
                    metadata={"seed": 99, "note": "reference writer"})
np.savez_compressed(os.path.join(HERE, "store_ref_values.npz"), times=times, values=values)
print("wrote store_ref.csv / store_ref.sdb1")
