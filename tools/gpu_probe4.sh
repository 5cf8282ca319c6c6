set -x
for c in C4 C2 C1; do
python tools/phases.py $c > gpurun_out/phases_$c.txt 2>&1
for rep in 1 2; do
python tools/prof_step.py $c 5 2>&1 | tail -1 | cut -c1-160 >> gpurun_out/inl_ab.txt
SK_LIB_PATH=$PWD/tools/ab/inl.so python tools/prof_step.py $c 5 2>&1 | tail -1 | cut -c1-160 >> gpurun_out/inl_ab.txt
done
done
