"""The bench's multi-rank (torchrun) path on one GPU: two ranks, each its
contiguous shard of the workload, gloo for the timing reductions
(SDEB200_BENCH_ONE_GPU=1 puts both on GPU 0).  Checks the strong-scaling
arithmetic of the JSON line rank 0 prints."""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_bench_line():
    env = dict(os.environ, SDEB200_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "cfg2", "--steps", "3",
           "--warmup", "3", "--no-cpu-baseline", "--no-cold"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["orbits_per_gpu"] == [32768]  # rank 0's half of cfg2
    # whole-job rate: all 65,536 orbits x 10^4 steps over the slowest rank's time
    assert abs(line["value"] - 65536 * 10000 / (line["ms_per_step"] * 1e-3)) < 1e-6 * line["value"]
    assert line["e2e"]["value"] > 0 and line["e2e"]["repeats_identical"]
