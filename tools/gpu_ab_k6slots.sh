#!/bin/bash
# K6 v4 split: 3-slot (default) vs 4-slot V ring
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6slots.log; : > $out
SSE_PI_V4_SLOTS=4 timeout 600 python -m pytest tests/test_gpu_pi.py -x -q -k "golden or split" > gpurun_out/r2_k6slots_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k6slots_tests.log
for rep in 1 2; do
  echo "3 slots: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "4 slots: $(SSE_PI_V4_SLOTS=4 timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
