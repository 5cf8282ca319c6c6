#!/bin/bash
# Interleaved A/B: tools/ab_run.sh CONFIG STEPS name1 name2 ... (libraries in tools/ab/;
# a name may carry environment settings: lib@VAR=val,VAR2=val)
cfg=$1; steps=$2; shift 2
for rep in 1 2; do
  for v in "$@"; do
    lib=${v%%@*}; envs=""; [[ $v == *@* ]] && envs=$(echo "${v#*@}" | tr ',' ' ')
    env $envs SK_LIB_PATH=$PWD/tools/ab/$lib.so timeout 300 python bench.py --config $cfg --steps $steps --warmup 5 --no-cpu-baseline > "gpurun_out/ab_${cfg}_${v}_$rep.log" 2>&1
  done
done
for v in "$@"; do for rep in 1 2; do
  python3 -c "
import json,sys; d=json.loads(open('gpurun_out/ab_${cfg}_${v}_$rep.log').read().strip().splitlines()[-1]); r=d['roofline']
print('$cfg $v $rep', '%.3e'%d['value'], 'ms %.3f'%d['ms_per_step'], {k:round(x,3) for k,x in r['stage_ms'].items()})"
done; done
