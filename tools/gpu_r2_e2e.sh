#!/bin/bash
# staging-ring tests + full default bench (e2e pageable + pinned, reference-atom parity)
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "staging or golden or kat" > gpurun_out/r2_pytest_staging.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_staging.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench2.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench2.log
