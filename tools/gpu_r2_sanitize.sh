#!/bin/bash
# momentum-group parity tests, then compute-sanitizer memcheck (one tool) on tiny K3m / phase calls
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multi_momentum or kernel_shapes" > gpurun_out/r2_mm_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_mm_tests.log
timeout 300 python tools/sanitize_small.py > gpurun_out/r2_sanitize_plain.log 2>&1 && \
  timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/r2_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/r2_memcheck.log
