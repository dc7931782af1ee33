#!/bin/bash
# round-2 evidence pass on the final commit: smoke, pytest -m gpu, default bench (N=1, all legs), the
# reference arm, small bench, staging trace (outputs small: no ncu here)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e9_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2e9_smoke.log
timeout 1800 python -m pytest tests -q -m gpu --durations=20 > gpurun_out/r2e9_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2e9_pytest_gpu.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r2e9_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2e9_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2e9_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2e9_bench_ref.log
timeout 600 python bench.py --config small --steps 5 --warmup 3 --no-e2e > gpurun_out/r2e9_bench_small.log 2>&1; echo "rc=$?" >> gpurun_out/r2e9_bench_small.log
SSE_STAGING_TRACE=1 timeout 900 python bench.py --steps 1 --warmup 3 --cpu-atoms 0 --pi-steps 0 --phase-device-steps 0 \
  --e2e-steps 2 --e2e-warmup 1 > gpurun_out/r2e9_trace.log 2>&1
echo "rc=$?" >> gpurun_out/r2e9_trace.log
