#!/bin/bash
TAG=${1:-p2e}
O=gpurun_out/$TAG
mkdir -p $O
export SDEB200_TUNE_CACHE=$PWD/$O/layouts.tsv
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 300 python tools/module_load_probe.py > $O/modload.log 2>&1; echo "modload rc=$?" >> $O/status.txt
for wl in cfg3_n256 paper_n15 cfg2 cfg1; do
  SDEB200_TRACE=1 SDEB200_TUNE_CACHE=$PWD/$O/cold_$wl.tsv timeout 300 python bench.py --cold-probe --workload $wl > $O/cold_$wl.log 2>&1; echo "cold $wl rc=$?" >> $O/status.txt
done
timeout 1800 python -m pytest tests -m gpu -q --tb=short --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
rm -f $SDEB200_TUNE_CACHE
timeout 900 python bench.py > $O/bench_cfg3.log 2>&1; echo "bench rc=$?" >> $O/status.txt
for wl in paper_n5 paper_n10 paper_n15; do
  timeout 400 python bench.py --workload $wl --coupling pairwise --no-cpu-baseline --no-cold --steps 3 > $O/bench_pw_$wl.log 2>&1; echo "bench pw $wl rc=$?" >> $O/status.txt
done
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 99 python tools/sanitize_cases.py autotune pairwise_lanes persistent > $O/memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/status.txt
