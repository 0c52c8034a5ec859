#!/bin/bash
TAG=${1:-p2i}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 900 python bench.py --no-cpu-baseline --no-cold > $O/bench_cfg3.log 2>&1; echo "bench rc=$?" >> $O/status.txt
for wl in cfg5 cfg1; do
  timeout 400 python bench.py --workload $wl --no-cpu-baseline --no-cold --steps 3 > $O/bench_$wl.log 2>&1; echo "bench $wl rc=$?" >> $O/status.txt
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kuramoto_run -c 1 -o $O/prof_n256 python tools/profile_run.py --workload cfg3_n256 --lanes 16 > $O/ncu_n256.log 2>&1; echo "ncu n256 rc=$?" >> $O/status.txt
python tools/ncu_summary.py $O/prof_n256.ncu-rep > $O/ncu_n256_summary.txt 2>&1
python tools/sass_exec_mix.py $O/prof_n256.ncu-rep > $O/ncu_n256_exec_mix.txt 2>&1
rm -f $O/prof_n256.ncu-rep
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --tb=short -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
