# Launch list + full capture of the widened-boundary kernels (assemble, transforms).
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/layer_launches.csv python tools/bench_layer.py > gpurun_out/layer_ncu.log 2>&1
for k in assemble_outer_kernel xform_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 -o gpurun_out/full_$k -f \
    python tools/bench_layer.py > gpurun_out/ncu_$k.log 2>&1
done
