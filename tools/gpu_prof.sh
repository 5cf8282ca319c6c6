# Phase probes + one full ncu capture of each solve kernel at C3 (run under gpurun).
mkdir -p gpurun_out
timeout 300 python tools/phases.py C3 > gpurun_out/phases_c3.txt 2>&1
timeout 300 python tools/phases.py C2 > gpurun_out/phases_c2.txt 2>&1
for k in theta_kernel lambda_fwd_kernel lambda_inv_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/full_$k -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
