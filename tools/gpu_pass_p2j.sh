#!/bin/bash
TAG=${1:-p2j}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 900 python -m pytest tests/test_gpu_bench_ranks.py -m gpu -q --tb=long > $O/pytest_ranks.log 2>&1; echo "pytest ranks rc=$?" >> $O/status.txt
for wl in cfg3_n256 paper_n5 paper_n15; do
  for rep in 1 2; do
    SDEB200_TRACE=1 SDEB200_TUNE_CACHE=$PWD/$O/cold_${wl}_$rep.tsv timeout 300 python bench.py --cold-probe --workload $wl > $O/cold_${wl}_$rep.log 2>&1; echo "cold $wl $rep rc=$?" >> $O/status.txt
  done
done
