#!/bin/bash
# Full GPU pass: smoke, GPU parity tests, headline bench (with CPU baseline),
# every workload, the ncu launch list of the headline bench and one
# `ncu --set full` capture of the cfg2 kernel at the autotuned layout.
# usage: bash tools/gpu_pass.sh TAG [workloads...]
TAG=${1:-pass}; shift
WLS=${@:-cfg1 cfg3_n32 cfg3_n64 cfg3_n128 cfg3_n256 cfg4 cfg5 cfg5_coherence cfg2_codegen ou_codegen paper_n5 paper_n10 paper_n15}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 900 python -m pytest tests -m gpu -q --tb=short --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_cfg2.log 2>&1; echo "bench rc=$?" >> $O/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.log 2>&1; echo "bench ref rc=$?" >> $O/status.txt
for wl in $WLS; do
  timeout 400 python bench.py --workload $wl --no-cpu-baseline --steps 3 > $O/bench_$wl.log 2>&1; echo "bench $wl rc=$?" >> $O/status.txt
done
timeout 300 python bench.py --coupling pairwise --no-cpu-baseline --steps 2 > $O/bench_cfg2_pairwise.log 2>&1; echo "bench pairwise rc=$?" >> $O/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> $O/status.txt
ARGS=$(python -c "import json;c=json.loads(open('$O/bench_cfg2.log').read().strip().splitlines()[-1])['config'];print('--lanes %d --persistent %d --ctas %d --tight %d --width %d' % (c['lanes_per_orbit'], c.get('persistent_grid',0), c.get('ctas_per_sm',0), c.get('register_capped',0), c.get('oscillators_per_lane',0)))" 2>/dev/null || echo "--lanes 2")
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kuramoto_run -c 1 -o $O/prof_cfg2 python tools/profile_run.py --workload cfg2 $ARGS > $O/ncu_full.log 2>&1; echo "ncu full rc=$? $ARGS" >> $O/status.txt
