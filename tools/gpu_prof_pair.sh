# Full GPU suite at HEAD + one full ncu capture of the C3 lambda kernels (run under gpurun).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests3.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests3.log
for k in lambda_fwd_pair_kernel lambda_inv_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/full_$k -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$k.log 2>&1
done
