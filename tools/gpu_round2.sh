# Round-2 measurement set on one B200 (run under gpurun); outputs in gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep -i "model name"
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
for c in C1 C2 C4 C5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err; done
timeout 900 python bench.py --gpus 2 --config C3 --steps 10 --warmup 3 > gpurun_out/r2_bench_c3_2ranks_1gpu.json 2> gpurun_out/r2_bench_2r.err
timeout 900 python tools/bench_coeff.py --c3 --out gpurun_out/r2_coeff_bench.json > gpurun_out/r2_coeff.log 2>&1
timeout 900 python tools/bench_layer.py > gpurun_out/r2_layer_bench.jsonl 2> gpurun_out/r2_layer.err
timeout 900 python tools/cufft_compare.py > gpurun_out/r2_cufft_compare.jsonl 2> gpurun_out/r2_cufft.err
# ncu: launch list of the bench command, then one full capture of the C3 theta kernel
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2_c3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:theta_sym -s 2 -c 1 -f -o gpurun_out/r2_theta_sym_c3 python tools/prof_step.py C3 2 > gpurun_out/r2_ncu_theta.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lambda_fwd_pair -s 2 -c 1 -f -o gpurun_out/r2_lambda_fwd_c3 python tools/prof_step.py C3 2 > gpurun_out/r2_ncu_lfwd.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
