#!/bin/bash
# Codegen pass: benches of the NVRTC-generated programs + one ncu capture.
TAG=${1:-codegen}
O=gpurun_out/$TAG
mkdir -p $O
for wl in cfg2_codegen ou_codegen; do
  timeout 600 python bench.py --workload $wl --steps 3 > $O/bench_$wl.log 2>&1; echo "bench $wl rc=$?" >> $O/status.txt
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sdb_dsl_main -c 1 -o $O/prof_cfg2_codegen python bench.py --workload cfg2_codegen --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_cfg2_codegen.log 2>&1; echo "ncu rc=$?" >> $O/status.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sdb_dsl_main -c 1 -o $O/prof_ou_codegen python bench.py --workload ou_codegen --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_ou_codegen.log 2>&1; echo "ncu ou rc=$?" >> $O/status.txt
