#!/bin/bash
# K5 with one CTA barrier per (point, polarity) step (double-buffered G2) vs HEAD; Pi parity
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_pi.py -x -q > gpurun_out/r2_k5_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k5_tests.log
out=gpurun_out/r2_ab_k5.log; : > $out
for rep in 1 2; do
  echo "head: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 --lib tools/ab/libsse_head.so 2>&1 | tail -1)" >> $out
  echo "new:  $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
