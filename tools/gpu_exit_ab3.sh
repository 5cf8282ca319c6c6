# C5 A/B of the relaxed cluster exit barrier (theta_large + lambda split kernels), the GPU suite, C3 bench with cpu_baseline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests6.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests6.log
timeout 900 python bench.py --config C5 --steps 5 --no-cpu-baseline > gpurun_out/exit3_c5_relaxed.json 2>> gpurun_out/exit3_ab.err
SK_PAIR_SYNC_EXIT=1 timeout 900 python bench.py --config C5 --steps 5 --no-cpu-baseline > gpurun_out/exit3_c5_sync.json 2>> gpurun_out/exit3_ab.err
timeout 600 python bench.py > gpurun_out/exit3_c3_full.json 2>> gpurun_out/exit3_ab.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3_b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
