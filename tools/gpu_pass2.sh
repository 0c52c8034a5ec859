#!/bin/bash
# Round-2 GPU pass: smoke, GPU tests, the default bench (cfg3 headline + cfg2
# secondary + cold call + reference CPU legs), the reference arm, autotune
# traces of the short-run shapes.
# usage: bash tools/gpu_pass2.sh TAG [skip-tests]
TAG=${1:-pass}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1; free -g > $O/free.txt 2>&1
export SDEB200_TUNE_CACHE=$PWD/$O/layouts.tsv
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
if [ "$2" != "skip-tests" ]; then
timeout 1500 python -m pytest tests -m gpu -q --tb=short --timeout 600 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
fi
rm -f $SDEB200_TUNE_CACHE
timeout 900 python bench.py > $O/bench_cfg3.log 2>&1; echo "bench rc=$?" >> $O/status.txt
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.log 2>&1; echo "bench ref rc=$?" >> $O/status.txt
for wl in paper_n15 cfg1 cfg3_n256; do
  SDEB200_TRACE=1 timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 3 > $O/bench_$wl.log 2>&1; echo "bench $wl rc=$?" >> $O/status.txt
done
