#!/bin/bash
# K6 v4 split: 4 CTAs/SM at 128 registers (spills, default) vs 3 CTAs/SM at 162 registers (no spills)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6minb.log; : > $out
SSE_PI_V4_MINB=3 timeout 600 python -m pytest tests/test_gpu_pi.py -x -q -k "split" > gpurun_out/r2_k6minb_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k6minb_tests.log
for rep in 1 2; do
  echo "minb4 4 slots: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "minb3 4 slots: $(SSE_PI_V4_MINB=3 timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "minb3 5 slots: $(SSE_PI_V4_MINB=3 SSE_PI_V4_SLOTS=5 timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
