"""Wall time of cfg5 (3.2 GiB store) through run_batch + write_store_bin vs the
streaming writer run_batch_to_file, and the order-parameter-only run.

    python tools/stream_file_bench.py [dir]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1908_03869_b200 as sdb  # noqa: E402
from paper_1908_03869_b200 import storage  # noqa: E402

out_dir = sys.argv[1] if len(sys.argv) > 1 else "/tmp"
w = bench.WORKLOADS["cfg5"]
model = bench.make_model(sdb, w)
batch = bench.make_batch(sdb, w, 0)
cfg = sdb.EngineConfig(dt=w["dt"], tspan=w["dt"] * w["steps"], ksteps=w["ksteps"],
                       orbits=w["orbits"], seed=20260809, stream=w["stream"],
                       max_store_bytes=1 << 40)
orbit_steps = w["orbits"] * w["steps"]
a, b = os.path.join(out_dir, "a.sdb1"), os.path.join(out_dir, "b.sdb1")
storage.run_batch_to_file(model, cfg, batch, b)  # warm
for rep in range(2):
    t0 = time.perf_counter()
    store = sdb.run_batch(model, cfg, batch)
    t1 = time.perf_counter()
    storage.write_store_bin(store, a)
    t2 = time.perf_counter()
    del store
    storage.run_batch_to_file(model, cfg, batch, b)
    t3 = time.perf_counter()
    print("run_batch %.1f ms + write_store_bin %.1f ms = %.1f ms | run_batch_to_file %.1f ms "
          "(%.3e orbit-steps/s) | file %.2f GB" % (1e3 * (t1 - t0), 1e3 * (t2 - t1),
                                                   1e3 * (t2 - t0), 1e3 * (t3 - t2),
                                                   orbit_steps / (t3 - t2),
                                                   os.path.getsize(b) / 1e9), flush=True)
print("identical:", open(a, "rb").read() == open(b, "rb").read())
os.remove(a)
os.remove(b)
