#!/bin/bash
# staging ramp from 25 atoms + balanced device chunks: tests + bench (no cpu leg, no Pi) with the trace
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_loop.py -x -q -k "staging or timing or sse_phase or golden_parity_all_variants or device_api or multi_momentum" > gpurun_out/r2_e2e3_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_e2e3_tests.log
SSE_STAGING_TRACE=1 timeout 900 python bench.py --steps 3 --warmup 3 --cpu-atoms 0 --pi-steps 0 --phase-device-steps 0 \
  --e2e-steps 2 --e2e-warmup 1 > gpurun_out/r2_e2e3_trace.log 2>&1
echo "rc=$?" >> gpurun_out/r2_e2e3_trace.log
