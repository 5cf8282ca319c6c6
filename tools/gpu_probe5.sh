set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "C5 or split or cluster or repeated" > gpurun_out/pytest_c5.log 2>&1
python tools/prof_step.py C5 2 2>&1 | tail -1 | cut -c1-200 > gpurun_out/c5_step.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:theta_mp -s 5 -c 5 --csv --log-file gpurun_out/c5_mp_launches.csv python tools/prof_step.py C5 1 > /dev/null 2>&1
