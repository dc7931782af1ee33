#!/bin/bash
# K5: real-embedding component swap by FSEL after LDS.128 (tools/ab/libsse_k5base.so) vs a per-lane
# address offset (two LDS.64, in-tree build); Pi GPU tests on the new build first
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k5swap.log; : > $out
timeout 900 python -m pytest tests/test_gpu_pi.py tests/test_loop.py -x -q -m gpu > gpurun_out/r2_k5swap_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k5swap_tests.log
for rep in 1 2; do
  echo "paper fsel: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 --lib tools/ab/libsse_k5base.so 2>&1 | tail -1)" >> $out
  echo "paper addr: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "small fsel: $(timeout 300 python tools/profile_pi.py --config small --atoms 256 --steps 2 --lib tools/ab/libsse_k5base.so 2>&1 | tail -1)" >> $out
  echo "small addr: $(timeout 300 python tools/profile_pi.py --config small --atoms 256 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
