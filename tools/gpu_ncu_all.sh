#!/bin/bash
# One `ncu --set full` capture per workload at its autotuned layout (the
# bench's own choice, read back from a short bench run), summaries only.
TAG=${1:-ncuall}; shift
WLS=${@:-cfg2 cfg3_n32 cfg3_n64 cfg3_n128 cfg3_n256 cfg4 cfg5 cfg1 paper_n5 paper_n10 paper_n15}
O=gpurun_out/$TAG
mkdir -p $O
# reports are summarised on the box and deleted (gpurun_out must stay < 64 MiB)
summarize() {
  python tools/ncu_summary.py $O/prof_$1.ncu-rep > $O/ncu_$1_summary.txt 2>&1
  python tools/sass_exec_mix.py $O/prof_$1.ncu-rep > $O/ncu_$1_exec_mix.txt 2>&1
  ncu -i $O/prof_$1.ncu-rep --page raw --csv > $O/ncu_$1_raw.csv 2>/dev/null
  rm -f $O/prof_$1.ncu-rep
}
for wl in $WLS; do
  timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-cold --steps 2 --warmup 3 > $O/bench_$wl.log 2>&1
  ARGS=$(python -c "import json;c=json.loads(open('$O/bench_$wl.log').read().strip().splitlines()[-1])['config'];print('--lanes %d --persistent %d --ctas %d --tight %d --width %d' % (c['lanes_per_orbit'], c.get('persistent_grid',0), c.get('ctas_per_sm',0), c.get('register_capped',0), c.get('oscillators_per_lane',0)))" 2>/dev/null || echo "--lanes 2")
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:kuramoto_run -c 1 -o $O/prof_$wl python tools/profile_run.py --workload $wl $ARGS > $O/ncu_$wl.log 2>&1
  echo "$wl ncu rc=$? $ARGS" >> $O/status.txt
  summarize $wl
done
for wl in cfg2_codegen ou_codegen cfg5_coherence; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sdb_dsl_main|kuramoto_run" -c 1 -o $O/prof_$wl python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-cold > $O/ncu_$wl.log 2>&1
  echo "$wl ncu rc=$?" >> $O/status.txt
  summarize $wl
done
