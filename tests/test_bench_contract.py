"""The bench.py contract parts that run without a GPU: the reference arm
(--impl reference) prints one JSON line with the required keys, and the
algorithmic FP64 counts stay consistent with the device code's operation
counts (DESIGN.md Roofline)."""

import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--workload", "cfg1", "--steps", "1", "--warmup", "1",
                          "--ref-seconds", "0.5"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    # the unmodified reference when baseline/_ref is installed, else the oracle port
    kind = "reference" if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "sdebatch")) \
        else "port"
    assert line["cpu_baseline"]["kind"] == kind and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["config"]["workload"] == "cfg1"


def test_reference_arm_defaults_to_the_headline_size():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.DEFAULT_WORKLOAD == "cfg3"
    assert bench.WORKLOADS["cfg3"]["headline"] == "cfg3_n256"
    w = bench.WORKLOADS["cfg3_n256"]
    assert (w["n"], w["orbits"], w["steps"], w["stream"]) == (256, 1 << 20, 100, "philox")


def test_shard_plans_are_contiguous_strong_splits():
    sys.path.insert(0, ROOT)
    import bench
    m = 1 << 20
    for gpus in (1, 2, 4, 8):
        plan = bench.plan_shards(m, 1, 0, 0, gpus)
        assert [d for d, _, _ in plan] == list(range(gpus))
        assert plan[0][1] == 0 and plan[-1][2] == m
        assert all(a[2] == b[1] for a, b in zip(plan, plan[1:]))
        ranks = [bench.plan_shards(m, gpus, r, r, gpus)[0] for r in range(gpus)]
        assert ranks == plan


def test_sharded_batches_equal_slices_of_the_whole():
    # the workload batch of a shard is exactly those rows of the whole batch
    # (global ids): host-side shaping checked with a stand-in sampler
    sys.path.insert(0, ROOT)
    import bench

    class B:
        def __init__(self, init, params):
            self.init, self.params = init, params

    def sample(count, omega, noise, k, first):
        ids = np.arange(first, first + count, dtype=np.float64)[:, None]
        return B(np.repeat(ids, 4, 1), np.repeat(ids * 10 + k, 9, 1))
    for kind in ("speed", "kgrid", "kgrid_ode", "resample"):
        w = dict(n=4, orbits=4096, batch=kind)
        whole = bench._shape_batch(B, w, 0, 4096, sample)
        for lo, hi in ((0, 1000), (1000, 2049), (2049, 4096), (300, 301)):
            part = bench._shape_batch(B, w, lo, hi, sample)
            assert np.array_equal(part.init, whole.init[lo:hi]), kind
            assert np.array_equal(part.params, whole.params[lo:hi]), kind


def test_algorithmic_counts():
    sys.path.insert(0, ROOT)
    import bench
    # meanfield em: sincos 14 + sums 2 + increment 2 + update 2 + Box-Muller 34 / 2,
    # and the two scaled sums per orbit
    assert bench.algorithmic_fp64_ops(16, "em", "meanfield") == 16 * (14 + 2 + 2 + 2 + 17) + 2
    assert bench.algorithmic_fp64_ops(8, "rk4", "meanfield") == 4 * (8 * 18 + 2) + 8 * 13
    assert bench.template_fp64_ops(4, "ou") == 4 * (2 + 1 + 17 + 4)
    assert bench.template_fp64_ops(16, "kuramoto_template", "pairwise") == \
        16 * 16 * 14 + 16 * (3 + 1 + 17 + 4)
    assert set(bench.WORKLOADS) >= {"cfg1", "cfg2", "cfg3_n32", "cfg3_n256", "cfg4", "cfg5",
                                    "cfg5_coherence", "cfg2_codegen", "ou_codegen"}
