#!/bin/bash
# Iteration pass: GPU tests, headline bench, one ncu capture of the cfg2 kernel.
# usage: bash tools/gpu_iter.sh TAG [extra bench workloads...]
TAG=${1:-iter}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --tb=short --timeout 300 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status_$TAG.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/status_$TAG.txt
for wl in "$@"; do
  timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 3 > gpurun_out/bench_${wl}_$TAG.log 2>&1; echo "bench $wl rc=$?" >> gpurun_out/status_$TAG.txt
done
LANES=$(python -c "import json;print(json.loads(open('gpurun_out/bench_cfg2_$TAG.log').read().strip().splitlines()[-1])['config']['lanes_per_orbit'])" 2>/dev/null || echo 4)
PROFARGS=$(python -c "import json;c=json.loads(open('gpurun_out/bench_cfg2_$TAG.log').read().strip().splitlines()[-1])['config'];print('--persistent %d --ctas %d' % (c.get('persistent_grid',0), c.get('ctas_per_sm',0)))" 2>/dev/null || echo "")
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kuramoto_run -c 1 -o gpurun_out/prof_cfg2_$TAG python tools/profile_run.py --workload cfg2 --steps 1000 --lanes $LANES $PROFARGS > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$? lanes=$LANES" >> gpurun_out/status_$TAG.txt
