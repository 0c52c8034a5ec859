#!/bin/bash
TAG=${1:-p2o}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
T0=$(date +%s); timeout 1200 python bench.py > $O/bench_default.log 2>&1; echo "bench rc=$? wall_s=$(( $(date +%s) - T0 ))" >> $O/status.txt
SDEB200_TRACE=1 timeout 900 python bench.py --no-cpu-baseline --no-cold > $O/bench_trace.log 2>&1; echo "bench trace rc=$?" >> $O/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_ranks.py -m gpu -q --tb=short > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
