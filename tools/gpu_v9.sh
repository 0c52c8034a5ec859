mkdir -p gpurun_out
python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2_$1.log 2>&1
for wl in cfg1 cfg3_n32 cfg3_n64 cfg3_n128 cfg3_n256 cfg4 cfg5; do python bench.py --workload $wl --no-cpu-baseline --steps 3 > gpurun_out/bench_${wl}_$1.log 2>&1; done
ncu --set full --import-source on --clock-control none -k regex:kuramoto_run -c 1 -o gpurun_out/prof_cfg2_$1 python tools/profile_run.py --workload cfg2 --steps 2000 --lanes 2 --persistent 1 > gpurun_out/ncu_$1.log 2>&1
