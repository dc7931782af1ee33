#!/bin/bash
# momentum-group parity tests, in-library multi-GPU path on one GPU, then compute-sanitizer memcheck
# (one tool) on tiny K3m / SSE-phase calls
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pi.py -q -k "multi_momentum or kernel_shapes or in_library or golden" > gpurun_out/r2_mm_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_mm_tests.log



