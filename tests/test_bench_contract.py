"""The bench.py contract parts that run without a GPU: the reference arm
(--impl reference) prints one JSON line with the required keys, and the
algorithmic FP64 counts stay consistent with the device code's operation
counts (DESIGN.md Roofline)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1", "--ref-seconds", "0.5"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["config"]["workload"] == "cfg2"


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
