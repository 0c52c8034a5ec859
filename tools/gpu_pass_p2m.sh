#!/bin/bash
TAG=${1:-p2m}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
T0=$(date +%s); timeout 1200 python bench.py > $O/bench_default.log 2>&1; echo "bench rc=$? wall_s=$(( $(date +%s) - T0 ))" >> $O/status.txt
T0=$(date +%s); timeout 1200 python bench.py --steps 20 --warmup 3 > $O/bench_default_k20.log 2>&1; echo "bench k20 rc=$? wall_s=$(( $(date +%s) - T0 ))" >> $O/status.txt
T0=$(date +%s); timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference_k20.log 2>&1; echo "bench ref k20 rc=$? wall_s=$(( $(date +%s) - T0 ))" >> $O/status.txt
