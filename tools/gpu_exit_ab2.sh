# A/B of the relaxed cluster exit barrier (lambda_fwd_pair + theta) at C3 and C4, plus the GPU suite.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests5.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests5.log
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/exit2_relaxed_$i.json 2>> gpurun_out/exit2_ab.err
  SK_PAIR_SYNC_EXIT=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/exit2_sync_$i.json 2>> gpurun_out/exit2_ab.err
done
timeout 600 python bench.py --config C4 --no-cpu-baseline > gpurun_out/exit2_c4_relaxed.json 2>> gpurun_out/exit2_ab.err
SK_PAIR_SYNC_EXIT=1 timeout 600 python bench.py --config C4 --no-cpu-baseline > gpurun_out/exit2_c4_sync.json 2>> gpurun_out/exit2_ab.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/exit2_c2_relaxed.json 2>> gpurun_out/exit2_ab.err
SK_PAIR_SYNC_EXIT=1 timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/exit2_c2_sync.json 2>> gpurun_out/exit2_ab.err
