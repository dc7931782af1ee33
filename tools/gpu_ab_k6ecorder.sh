#!/bin/bash
# K6 grid order: the short last E-chunk's main CTAs interleaved (tools/ab/libsse_base.so) vs last in
# the main grid (in-tree build); Pi tests first (bitwise equal variants, goldens)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6ecorder.log; : > $out
timeout 900 python -m pytest tests/test_gpu_pi.py -x -q > gpurun_out/r2_k6ecorder_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k6ecorder_tests.log
for rep in 1 2; do
  echo "interleaved: $(timeout 300 python tools/profile_pi.py --atoms 196 --steps 1 --lib tools/ab/libsse_base.so 2>&1 | tail -1)" >> $out
  echo "short last:  $(timeout 300 python tools/profile_pi.py --atoms 196 --steps 1 2>&1 | tail -1)" >> $out
done
cat $out
