#!/bin/bash
# module-load probe, J=16 register-capped layouts vs the natural ones, the
# default bench, sanitizer over every variant (incl. the new pairwise tiles).
TAG=${1:-p2b}
O=gpurun_out/$TAG
mkdir -p $O
export SDEB200_TUNE_CACHE=$PWD/$O/layouts.tsv
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 300 python tools/module_load_probe.py > $O/modload_lazy.log 2>&1; echo "modload lazy rc=$?" >> $O/status.txt
CUDA_MODULE_LOADING=EAGER timeout 300 python tools/module_load_probe.py > $O/modload_eager.log 2>&1; echo "modload eager rc=$?" >> $O/status.txt
for wl in cfg3_n256:16 cfg3_n128:8 cfg3_n64:4 cfg3_n32:2 cfg5:2; do
  name=${wl%%:*}; L=${wl##*:}
  for tight in 0 1; do
    SDEB200_LAYOUT=$L,0,0,$tight timeout 300 python bench.py --workload $name --no-cpu-baseline --no-cold --steps 3 > $O/bench_${name}_t$tight.log 2>&1; echo "bench $name tight=$tight rc=$?" >> $O/status.txt
  done
done
rm -f $SDEB200_TUNE_CACHE
timeout 900 python bench.py > $O/bench_cfg3.log 2>&1; echo "bench rc=$?" >> $O/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kuramoto_run -c 1 -o $O/prof_n256_tight python tools/profile_run.py --workload cfg3_n256 --lanes 16 --tight 1 > $O/ncu_n256_tight.log 2>&1; echo "ncu n256 tight rc=$?" >> $O/status.txt
python tools/ncu_summary.py $O/prof_n256_tight.ncu-rep > $O/ncu_n256_tight_summary.txt 2>&1
python tools/sass_exec_mix.py $O/prof_n256_tight.ncu-rep > $O/ncu_n256_tight_exec_mix.txt 2>&1
ncu -i $O/prof_n256_tight.ncu-rep --page raw --csv > $O/ncu_n256_tight_raw.csv 2>/dev/null
rm -f $O/prof_n256_tight.ncu-rep
bash tools/gpu_sanitize.sh $TAG/san
