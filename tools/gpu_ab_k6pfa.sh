#!/bin/bash
# K6 v4 split: default vs an L2 prefetch of the G1 rows one stage further ahead (SSE_PI_PFA=1);
# bitwise check of the Pi tests under the switch first
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6pfa.log; : > $out
SSE_PI_PFA=1 timeout 900 python -m pytest tests/test_gpu_pi.py -x -q -k "split or shapes" > gpurun_out/r2_k6pfa_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k6pfa_tests.log
for rep in 1 2; do
  echo "default: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "pfa:     $(SSE_PI_PFA=1 timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
