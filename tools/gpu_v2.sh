#!/bin/bash
# compare Sigma kernel variants (simple vs register-pipelined) + parity
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for K in 0 1; do SSE_SIGMA_KERNEL=$K timeout 300 python tools/profile_sigma.py --atoms 148 > gpurun_out/prof_k$K.log 2>&1; echo "K=$K rc=$?" >> gpurun_out/prof_k$K.log; done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
cat gpurun_out/prof_k0.log gpurun_out/prof_k1.log; tail -3 gpurun_out/pytest_gpu.log
