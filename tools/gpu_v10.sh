mkdir -p gpurun_out
python -m pytest tests -m gpu -q --tb=short --timeout 300 > gpurun_out/pytest_gpu_$1.log 2>&1
python tools/layout_sweep.py --workload cfg2 > gpurun_out/sweep_cfg2_$1.log 2>&1
python tools/layout_sweep.py --workload cfg3_n32 > gpurun_out/sweep_cfg3_n32_$1.log 2>&1
python tools/e2e_breakdown.py --workload cfg2 > gpurun_out/e2e_cfg2_$1.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2_$1.log 2>&1
