#!/bin/bash
TAG=${1:-p2n}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
for wl in cfg5 cfg5_coherence cfg4 paper_n15; do
  timeout 400 python bench.py --workload $wl --no-cpu-baseline --no-cold --steps 3 > $O/bench_$wl.log 2>&1; echo "bench $wl rc=$?" >> $O/status.txt
done
timeout 900 python bench.py --no-cpu-baseline --no-cold > $O/bench_cfg3.log 2>&1; echo "bench rc=$?" >> $O/status.txt
timeout 1800 python -m pytest tests -m gpu -q --tb=short --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
