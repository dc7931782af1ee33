#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/fp64_mixed tools/microbench/fp64_mixed.cu && \
  timeout 120 ./tools/microbench/fp64_mixed > gpurun_out/fp64_mixed.txt 2>&1; cat gpurun_out/fp64_mixed.txt
bash tools/gpu_ncu_pi.sh
