#!/bin/bash
# K6 v4 split: incremental counters (tools/ab/libsse_incr.so) vs + static A offsets with the
# stage-crossing sub-stage specialised (in-tree build); Pi GPU tests on the new build first
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6lastj.log; : > $out
timeout 900 python -m pytest tests/test_gpu_pi.py -x -q > gpurun_out/r2_k6lastj_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k6lastj_tests.log
for rep in 1 2; do
  echo "incr: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 --lib tools/ab/libsse_incr.so 2>&1 | tail -1)" >> $out
  echo "lastj: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
