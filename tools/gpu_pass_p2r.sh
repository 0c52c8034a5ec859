#!/bin/bash
# ncu --set full of the pairwise stepper at cfg3 n=256 (L=32, J=8) and n=32 (L=4, J=8)
TAG=${1:-p2r}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for spec in cfg3_n256:32 cfg3_n32:4; do
  wl=${spec%%:*}; L=${spec##*:}
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:kuramoto_run -c 1 -o $O/prof_pw_$wl python tools/profile_run.py --workload $wl --coupling pairwise --lanes $L > $O/ncu_pw_$wl.log 2>&1; echo "ncu pw $wl rc=$?" >> $O/status.txt
  python tools/ncu_summary.py $O/prof_pw_$wl.ncu-rep > $O/ncu_pw_${wl}_summary.txt 2>&1
  python tools/sass_exec_mix.py $O/prof_pw_$wl.ncu-rep > $O/ncu_pw_${wl}_exec_mix.txt 2>&1
  rm -f $O/prof_pw_$wl.ncu-rep
done
