#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for K in 1 2 0; do SSE_SIGMA_KERNEL=$K timeout 300 python tools/profile_sigma.py --atoms 148 > gpurun_out/prof_k$K.log 2>&1; echo "K=$K rc=$?" >> gpurun_out/prof_k$K.log; cat gpurun_out/prof_k$K.log; done
SSE_SIGMA_KERNEL=2 timeout 900 python -m pytest tests -x -q -m gpu -k "not paper_config" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
