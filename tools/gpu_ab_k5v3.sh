#!/bin/bash
# K5 v3 (barrier-free, V stored straight to HBM; SSE_PI_BUILD=3) vs K5 v2: parity + A/B
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
SSE_PI_BUILD=3 timeout 900 python -m pytest tests/test_gpu_pi.py tests/test_loop.py -x -q -m gpu > gpurun_out/r2_k5v3_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k5v3_tests.log
out=gpurun_out/r2_ab_k5v3.log; : > $out
for rep in 1 2; do
  echo "v2: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "v3: $(SSE_PI_BUILD=3 timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
