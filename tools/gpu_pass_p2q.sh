#!/bin/bash
TAG=${1:-p2q}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 1800 python -m pytest tests -m gpu -q --tb=short --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
T0=$(date +%s); timeout 1200 python bench.py > $O/bench_default.log 2>&1; echo "bench rc=$? wall_s=$(( $(date +%s) - T0 ))" >> $O/status.txt
T0=$(date +%s); timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1; echo "bench ref rc=$? wall_s=$(( $(date +%s) - T0 ))" >> $O/status.txt
for wl in paper_n15 cfg2; do
  SDEB200_TRACE=1 SDEB200_TUNE_CACHE=$PWD/$O/cold_${wl}.tsv timeout 300 python bench.py --cold-probe --workload $wl > $O/cold_${wl}.log 2>&1; echo "cold $wl rc=$?" >> $O/status.txt
done
