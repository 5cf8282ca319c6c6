timeout 900 python -m pytest tests -m gpu -q -x -k "coeff or kat or residual or exact or cli or abi or integration or bench_poisson" > gpurun_out/pytest_k5.log 2>&1
python tools/bench_coeff.py --sizes 512,1024,2048,4096 --c3 --no-ref --out gpurun_out/r2_coeff_bench_new.json > gpurun_out/k5.log 2>&1
