#!/bin/bash
TAG=${1:-p2h}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
SDEB200_TRACE=1 timeout 900 python bench.py --no-cpu-baseline --no-cold > $O/bench_cfg3.log 2>&1; echo "bench rc=$?" >> $O/status.txt
for wl in cfg4 cfg5 paper_n15 paper_n5 cfg1; do
  SDEB200_TRACE=1 timeout 400 python bench.py --workload $wl --no-cpu-baseline --no-cold --steps 3 > $O/bench_$wl.log 2>&1; echo "bench $wl rc=$?" >> $O/status.txt
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --tb=short -k "autotune or layout or pinned or shards" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
