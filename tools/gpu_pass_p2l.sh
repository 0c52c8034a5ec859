#!/bin/bash
TAG=${1:-p2l}
O=gpurun_out/$TAG
mkdir -p $O
for wl in cfg3_n256 paper_n15 paper_n5 cfg2; do
  SDEB200_TRACE=1 SDEB200_TUNE_CACHE=$PWD/$O/cold_${wl}.tsv timeout 300 python bench.py --cold-probe --workload $wl > $O/cold_${wl}.log 2>&1; echo "cold $wl rc=$?" >> $O/status.txt
done
timeout 1200 python bench.py > $O/bench_default.log 2>&1; echo "bench rc=$?" >> $O/status.txt
timeout 1800 python -m pytest tests -m gpu -q --tb=short --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
