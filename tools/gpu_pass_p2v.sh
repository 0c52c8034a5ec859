#!/bin/bash
# stage-2 tuning at the run's own length: GPU tests, default bench, traced n=256 tune
TAG=${1:-p2v}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 1800 python -m pytest tests -m gpu -q --tb=short --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
T0=$(date +%s); timeout 1200 python bench.py > $O/bench_default.log 2>&1; echo "bench rc=$? wall_s=$(( $(date +%s) - T0 ))" >> $O/status.txt
SDEB200_TRACE=1 timeout 300 python bench.py --workload cfg3_n256 --no-cold --no-secondary --no-cpu-baseline --steps 10 > $O/bench_n256_trace.log 2>&1; echo "n256 trace rc=$?" >> $O/status.txt
