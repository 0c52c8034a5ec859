#!/bin/bash
# First GPU pass: smoke, GPU parity tests, bench, ncu launch list + full capture.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -q --tb=short --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
for wl in cfg1 cfg3_n32 cfg3_n256 cfg4 cfg5; do
  timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 3 > gpurun_out/bench_$wl.log 2>&1; echo "bench $wl rc=$?" >> gpurun_out/status.txt
done
timeout 300 python bench.py --coupling pairwise --no-cpu-baseline --steps 2 > gpurun_out/bench_cfg2_pairwise.log 2>&1; echo "bench pairwise rc=$?" >> gpurun_out/status.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/status.txt
LANES=$(python -c "import json;print(json.loads(open('gpurun_out/bench_cfg2.log').read().strip().splitlines()[-1])['config']['lanes_per_orbit'])" 2>/dev/null || echo 2)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kuramoto_run -c 1 -o gpurun_out/prof_cfg2 python tools/profile_run.py --workload cfg2 --steps 1000 --lanes $LANES > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$? lanes=$LANES" >> gpurun_out/status.txt
