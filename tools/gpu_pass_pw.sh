#!/bin/bash
# Pairwise + cold-call pass: GPU tests, pairwise benches (cfg2, cfg3 sizes),
# cold-call traces, ncu of the pairwise kernel.
# usage: bash tools/gpu_pass_pw.sh TAG
TAG=${1:-pw}
O=gpurun_out/$TAG
mkdir -p $O
export SDEB200_TUNE_CACHE=$PWD/$O/layouts.tsv
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 1800 python -m pytest tests -m gpu -q --tb=short --timeout 900 -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
for wl in cfg3_n256 paper_n15 cfg1; do
  SDEB200_TRACE=1 SDEB200_TUNE_CACHE=$PWD/$O/cold_$wl.tsv timeout 300 python bench.py --cold-probe --workload $wl > $O/cold_$wl.log 2>&1; echo "cold $wl rc=$?" >> $O/status.txt
done
for wl in cfg2 cfg3_n32 cfg3_n64 cfg3_n128 cfg3_n256 paper_n15; do
  timeout 600 python bench.py --workload $wl --coupling pairwise --no-cpu-baseline --no-cold --steps 3 > $O/bench_pw_$wl.log 2>&1; echo "bench pw $wl rc=$?" >> $O/status.txt
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kuramoto_run -c 1 -o $O/prof_pw_cfg2 python tools/profile_run.py --workload cfg2 --coupling pairwise --lanes 2 --steps 2000 > $O/ncu_pw_cfg2.log 2>&1; echo "ncu pw cfg2 rc=$?" >> $O/status.txt
python tools/ncu_summary.py $O/prof_pw_cfg2.ncu-rep > $O/ncu_pw_cfg2_summary.txt 2>&1
python tools/sass_exec_mix.py $O/prof_pw_cfg2.ncu-rep > $O/ncu_pw_cfg2_exec_mix.txt 2>&1
rm -f $O/prof_pw_cfg2.ncu-rep
