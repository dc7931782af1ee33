#!/bin/bash
# K6 v4 split (3 CTAs / SM): stage counters recomputed from ss (tools/ab/libsse_head.so) vs
# incremental counters (in-tree build); bitwise tests on the new build first
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6incr.log; : > $out
timeout 900 python -m pytest tests/test_gpu_pi.py -x -q > gpurun_out/r2_k6incr_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k6incr_tests.log
for rep in 1 2; do
  echo "head: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 --lib tools/ab/libsse_head.so 2>&1 | tail -1)" >> $out
  echo "incr: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
