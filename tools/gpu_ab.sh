# usage: bash tools/gpu_ab.sh "CONFIGS" name1 name2 ...   (tests run on the in-tree library first)
mkdir -p gpurun_out
cfgs=$1; shift
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for c in $cfgs; do bash tools/ab_run.sh $c 10 "$@"; done
