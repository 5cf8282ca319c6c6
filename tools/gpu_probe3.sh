set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "theta_sym or full_size_analytic or lambda or golden or rough" > gpurun_out/pytest_sym.log 2>&1
python tools/phases.py C3 > gpurun_out/phases_c3.txt 2>&1
python tools/size_probe.py 20000 10000 10 > gpurun_out/size_probe.txt 2>&1
SK_LAMBDA_DUO=0 python tools/size_probe.py 20000 10000 10 >> gpurun_out/size_probe.txt 2>&1
