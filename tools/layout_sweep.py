"""Time a bench workload at pinned launch layouts (lanes, persistent, ctas/SM).

    python tools/layout_sweep.py --workload cfg2 [--steps N]

Each layout runs in a fresh process-level context (SDEB200_LAYOUT pinned) so
the autotuner is bypassed; prints ms per full run (CUDA events, best of 3).
"""

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1908_03869_b200 as sdb  # noqa: E402
from paper_1908_03869_b200 import _native as nat  # noqa: E402
from paper_1908_03869_b200.engine import make_desc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--layouts", default="")
    args = ap.parse_args()
    w = dict(bench.WORKLOADS[args.workload])
    if args.steps:
        w["steps"] = args.steps
        w["ksteps"] = min(w["ksteps"], args.steps)
    n, m, steps = w["n"], w["orbits"], w["steps"]
    chunks = steps // w["ksteps"]
    p = 1
    while p < n:
        p *= 2
    lanes_opts = [L for L in (1, 2, 4, 8, 16, 32) if L <= p and p // L <= 16]
    layouts = ([tuple(int(x) for x in s.split(",")) for s in args.layouts.split(";")]
               if args.layouts else
               [(L, pers, 0, tight) for L in lanes_opts for pers in (0, 1)
                for tight in ((0, 1) if (p // L) in (4, 8) and p == n else (0,))])
    model = bench.make_model(sdb, w)
    batch = bench.make_batch(sdb, w, 0)
    cfg = sdb.EngineConfig(dt=w["dt"], tspan=w["dt"] * steps, ksteps=w["ksteps"], orbits=m,
                           solver=w["solver"], seed=20260809, stream=w["stream"],
                           max_store_bytes=1 << 40)
    desc = make_desc(model, cfg, chunks, m)
    d_init = torch.from_numpy(np.ascontiguousarray(batch.init)).cuda()
    d_params = torch.from_numpy(np.ascontiguousarray(batch.params)).cuda()
    d_values = torch.empty((m, chunks, n), dtype=torch.float64, device="cuda")
    d_fail = torch.empty(m, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    lib = nat.lib()
    ref = None
    for lay in layouts:
        os.environ["SDEB200_LAYOUT"] = ",".join(str(v) for v in lay)
        ctx = ctypes.c_void_p()
        nat.check(lib.sdb_open(None, 0, ctypes.byref(ctx)))
        times = []
        for rep in range(4):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            nat.check(lib.sdb_run_device(ctx, desc, d_init.data_ptr(), d_params.data_ptr(),
                                         d_values.data_ptr(), d_fail.data_ptr(),
                                         stream.cuda_stream), ctx)
            e1.record(stream)
            torch.cuda.synchronize()
            if rep:
                times.append(e0.elapsed_time(e1))
        out = d_values.cpu().numpy()
        same = ref is None or np.array_equal(out, ref, equal_nan=True)
        if ref is None:
            ref = out
        got = [ctypes.c_int32() for _ in range(5)]
        lib.sdb_last_layout(ctx, *(ctypes.byref(v) for v in got))
        print(json.dumps({"layout": lay, "ran": [v.value for v in got], "ms": min(times),
                          "orbit_steps_per_s": m * steps / (min(times) * 1e-3),
                          "bitwise_same": bool(same)}), flush=True)
        lib.sdb_close(ctx)


if __name__ == "__main__":
    main()
