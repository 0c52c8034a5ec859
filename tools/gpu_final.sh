#!/bin/bash
# Round-2 final pass: smoke, GPU tests, the default bench (cfg3 + cfg2, CPU legs
# from the reference, cold call), the reference arm, every workload (meanfield
# and pairwise), the ncu launch list of the default bench, one ncu --set full
# capture per workload, the sanitizer suite.
TAG=${1:-final}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1; free -g > $O/free.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 1800 python -m pytest tests -m gpu -q --tb=short --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
T0=$(date +%s); timeout 1200 python bench.py > $O/bench_default.log 2>&1; echo "bench rc=$? wall_s=$(( $(date +%s) - T0 ))" >> $O/status.txt
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.log 2>&1; echo "bench ref rc=$?" >> $O/status.txt
for wl in cfg1 cfg4 cfg5 cfg5_coherence paper_n5 paper_n10 paper_n15 cfg2_codegen ou_codegen; do
  timeout 400 python bench.py --workload $wl --no-cpu-baseline --steps 3 > $O/bench_$wl.log 2>&1; echo "bench $wl rc=$?" >> $O/status.txt
done
for wl in cfg2 cfg3_n32 cfg3_n64 cfg3_n128 cfg3_n256 paper_n5 paper_n10 paper_n15; do
  timeout 600 python bench.py --workload $wl --coupling pairwise --no-cpu-baseline --no-cold --steps 3 > $O/bench_pw_$wl.log 2>&1; echo "bench pw $wl rc=$?" >> $O/status.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cold > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> $O/status.txt
bash tools/gpu_ncu_all.sh $TAG/ncu
bash tools/gpu_sanitize.sh $TAG/san
