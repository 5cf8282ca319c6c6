# A/B of the lambda_fwd_pair exit barrier (relaxed arrive vs cluster.sync) at C3, plus the GPU suite.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests4.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests4.log
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/exit_relaxed_$i.json 2>> gpurun_out/exit_ab.err
  SK_PAIR_SYNC_EXIT=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/exit_sync_$i.json 2>> gpurun_out/exit_ab.err
done
