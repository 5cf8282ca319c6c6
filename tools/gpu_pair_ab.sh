mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "row_pairs" > gpurun_out/pair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pair_tests.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests2.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests2.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_pair.json 2> gpurun_out/bench_c3_pair.err
SK_LAMBDA_PAIR_INV=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_nopair.json 2>> gpurun_out/bench_c3_pair.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_pair2.json 2>> gpurun_out/bench_c3_pair.err
