#!/bin/bash
# Host-pipeline pass: GPU tests, e2e breakdowns with per-phase trace, bench
# lines for the I/O-heavy workloads, ncu of the benched cfg2 kernel (full run).
TAG=${1:-e2e}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --tb=short --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
for wl in cfg2 cfg5 cfg3_n32 cfg3_n256; do
  SDEB200_TRACE=1 timeout 300 python tools/e2e_breakdown.py --workload $wl --reps 3 > $O/e2e_$wl.log 2>&1; echo "e2e $wl rc=$?" >> $O/status.txt
done
timeout 600 python bench.py --no-cpu-baseline > $O/bench_cfg2.log 2>&1; echo "bench rc=$?" >> $O/status.txt
for wl in cfg5 cfg3_n32 cfg3_n256; do
  timeout 400 python bench.py --workload $wl --no-cpu-baseline --steps 3 > $O/bench_$wl.log 2>&1; echo "bench $wl rc=$?" >> $O/status.txt
done
ARGS=$(python -c "import json;c=json.loads(open('$O/bench_cfg2.log').read().strip().splitlines()[-1])['config'];print('--lanes %d --persistent %d --ctas %d --tight %d --width %d' % (c['lanes_per_orbit'], c.get('persistent_grid',0), c.get('ctas_per_sm',0), c.get('register_capped',0), c.get('oscillators_per_lane',0)))" 2>/dev/null || echo "--lanes 4")
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kuramoto_run -c 1 -o $O/prof_cfg2 python tools/profile_run.py --workload cfg2 $ARGS > $O/ncu_full.log 2>&1; echo "ncu full rc=$? $ARGS" >> $O/status.txt
