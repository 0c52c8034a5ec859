"""Where the end-to-end run_batch time goes (host staging vs kernel).

    python tools/e2e_breakdown.py --workload cfg2
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1908_03869_b200 as sdb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    w = bench.WORKLOADS[args.workload]
    n, m, steps = w["n"], w["orbits"], w["steps"]
    model = bench.make_model(sdb, w)
    batch = bench.make_batch(sdb, w, 0)
    cfg = sdb.EngineConfig(dt=w["dt"], tspan=w["dt"] * steps, ksteps=w["ksteps"], orbits=m,
                           solver=w["solver"], seed=20260809, stream=w["stream"],
                           max_store_bytes=1 << 40)
    sdb.run_batch(model, cfg, batch)  # warm: autotune + buffers
    t = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        sdb.run_batch(model, cfg, batch)
        t.append(time.perf_counter() - t0)
    chunks = steps // w["ksteps"]
    t_alloc = time.perf_counter()
    v = np.empty((m, chunks + 1, n))
    v[:] = 0.0
    t_alloc = time.perf_counter() - t_alloc
    print("run_batch e2e: best %.2f ms, median %.2f ms" % (1e3 * min(t), 1e3 * np.median(t)))
    print("first-touch of a fresh (M, k+1, n) store: %.2f ms (%.1f MB)" % (1e3 * t_alloc, v.nbytes / 1e6))
    print("input bytes %.1f MB, output bytes %.1f MB" % ((batch.init.nbytes + batch.params.nbytes) / 1e6,
                                                        m * chunks * n * 8 / 1e6))


if __name__ == "__main__":
    main()
