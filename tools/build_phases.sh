#!/bin/bash
# Debug build of the library with the theta-kernel phase probes (-DSK_PHASES).
set -e
cd "$(dirname "$0")/.."
mkdir -p /tmp/phasebuild
pids=()
for f in grid_kernels grid_large theta_sym theta_mp lambda_duo coeff_kernels assemble_kernels ge_kernels transforms sk_poisson; do
  extra=""; case $f in coeff_kernels|assemble_kernels|ge_kernels) extra="--fmad=false";; esac
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -rdc=true -DSK_PHASES -DSK_CHAIN_ATTR=__forceinline__ -Xcompiler -fPIC $extra \
       -Iinclude -c paper_1510_08094_b200/csrc/$f.cu -o /tmp/phasebuild/$f.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
nvcc -gencode arch=compute_100a,code=sm_100a -rdc=true -shared -cudart static -o tools/libsk_poisson_phases.so /tmp/phasebuild/*.o
