#!/bin/bash
# K5 DMMA build for No = 10 (padded split K): Pi parity + small-config bench
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_pi.py tests/test_loop.py -x -q -m gpu > gpurun_out/r2_k5no10_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k5no10_tests.log
timeout 600 python bench.py --config small --steps 5 --warmup 3 --no-e2e > gpurun_out/r2_k5no10_small.log 2>&1; echo "rc=$?" >> gpurun_out/r2_k5no10_small.log
