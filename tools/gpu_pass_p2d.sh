#!/bin/bash
# revert check + cold-call study + ncu of every workload (traffic.json).
TAG=${1:-p2d}
O=gpurun_out/$TAG
mkdir -p $O
export SDEB200_TUNE_CACHE=$PWD/$O/layouts.tsv
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 1800 python -m pytest tests -m gpu -q --tb=short --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
rm -f $SDEB200_TUNE_CACHE
timeout 900 python bench.py > $O/bench_cfg3.log 2>&1; echo "bench rc=$?" >> $O/status.txt
for wl in cfg3_n256 paper_n15 cfg1 cfg2; do
  SDEB200_TRACE=1 SDEB200_TUNE_CACHE=$PWD/$O/cold_$wl.tsv timeout 300 python bench.py --cold-probe --workload $wl > $O/cold_$wl.log 2>&1; echo "cold $wl rc=$?" >> $O/status.txt
  SDEB200_PIECE_KB=16384 SDEB200_TRACE=1 SDEB200_TUNE_CACHE=$PWD/$O/cold16_$wl.tsv timeout 300 python bench.py --cold-probe --workload $wl > $O/cold16_$wl.log 2>&1; echo "cold16 $wl rc=$?" >> $O/status.txt
done
SDEB200_PIECE_KB=16384 timeout 600 python bench.py --workload cfg3_n256 --no-cpu-baseline --no-cold --steps 3 > $O/bench_n256_piece16.log 2>&1; echo "bench piece16 rc=$?" >> $O/status.txt
timeout 600 python bench.py --workload cfg3_n256 --no-cpu-baseline --no-cold --steps 3 > $O/bench_n256_piece64.log 2>&1; echo "bench piece64 rc=$?" >> $O/status.txt
bash tools/gpu_ncu_all.sh $TAG/ncu
