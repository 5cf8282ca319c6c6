# per-kernel time / DRAM bytes / occupancy of the multi-pass theta stage at C5
python tools/prof_step.py C5 1 > gpurun_out/c5plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,smsp__inst_executed.sum --clock-control none -k regex:theta_mp -c 5 --csv --log-file gpurun_out/mp_launches.csv python tools/prof_step.py C5 1 > gpurun_out/ncu_mp.log 2>&1
