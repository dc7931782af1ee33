#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for K in 3 1; do SSE_SIGMA_KERNEL=$K timeout 300 python tools/profile_sigma.py --atoms 148 > gpurun_out/prof_k$K.log 2>&1; echo "K=$K rc=$?" >> gpurun_out/prof_k$K.log; cat gpurun_out/prof_k$K.log; done
