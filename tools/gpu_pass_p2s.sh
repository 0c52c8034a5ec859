#!/bin/bash
# ncu --set full of the pairwise stepper at cfg3 n=256 (L=32, J=8), step-shortened run
TAG=${1:-p2s}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
wl=cfg3_n256
timeout 1100 ncu --set full --import-source on --clock-control none -k regex:kuramoto_run -c 1 -o $O/prof_pw_$wl python tools/profile_run.py --workload $wl --coupling pairwise --lanes 32 --steps 8 > $O/ncu_pw_$wl.log 2>&1; echo "ncu pw $wl rc=$?" >> $O/status.txt
python tools/ncu_summary.py $O/prof_pw_$wl.ncu-rep > $O/ncu_pw_${wl}_summary.txt 2>&1
python tools/sass_exec_mix.py $O/prof_pw_$wl.ncu-rep > $O/ncu_pw_${wl}_exec_mix.txt 2>&1
rm -f $O/prof_pw_$wl.ncu-rep
