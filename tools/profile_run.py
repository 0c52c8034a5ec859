"""One device-resident run of a bench workload, for ncu captures.

    ncu --set full --import-source on -k regex:kuramoto_run -c 1 -o prof \
        python tools/profile_run.py --workload cfg2 --steps 2000 --lanes 2

--lanes pins the layout (no autotune probes in the capture); --steps
shortens the run (per-step work is identical, so counters per orbit-step
are unchanged).
"""

import argparse
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
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--coupling", default="meanfield")
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--persistent", type=int, default=0)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--tight", type=int, default=0)
    ap.add_argument("--width", type=int, default=0, help="oscillators per lane (exact layouts)")
    args = ap.parse_args()
    if args.lanes:
        os.environ["SDEB200_LAYOUT"] = "%d,%d,%d,%d,%d" % (args.lanes, args.persistent, args.ctas,
                                                           args.tight, args.width)
    w = dict(bench.WORKLOADS[args.workload])
    if args.steps:
        w["steps"] = args.steps
        w["ksteps"] = min(w["ksteps"], args.steps)
    n, m, steps = w["n"], w["orbits"], w["steps"]
    chunks = steps // w["ksteps"]
    model = bench.make_model(sdb, w)
    batch = bench.make_batch(sdb, w, 0)
    cfg = sdb.EngineConfig(dt=w["dt"], tspan=w["dt"] * steps, ksteps=w["ksteps"], orbits=m,
                           solver=w["solver"], seed=20260809, stream=w["stream"],
                           coupling=args.coupling, lanes=args.lanes, max_store_bytes=1 << 40)
    desc = make_desc(model, cfg, chunks, m)
    ctx = nat.context((0,))
    d_init = torch.from_numpy(np.ascontiguousarray(batch.init)).cuda()
    d_params = torch.from_numpy(np.ascontiguousarray(batch.params)).cuda()
    d_values = torch.empty((m, chunks, n), dtype=torch.float64, device="cuda")
    d_fail = torch.empty(m, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(args.repeat):
        nat.check(nat.lib().sdb_run_device(ctx, desc, d_init.data_ptr(), d_params.data_ptr(),
                                           d_values.data_ptr(), d_fail.data_ptr(),
                                           stream.cuda_stream), ctx)
    torch.cuda.synchronize()
    print("lanes", nat.lib().sdb_last_lanes(ctx), "finite", bool(torch.isfinite(d_values).all()))


if __name__ == "__main__":
    main()
