#!/bin/bash
# A/B of the Pi kernels on a 96-atom paper shard: HEAD build (tools/ab/libsse_head.so) vs the in-tree build
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
out=gpurun_out/ab_pi.log; : > $out
for rep in 1 2; do
  echo "head: $(timeout 300 python tools/profile_pi.py --atoms 96 --steps 2 --lib tools/ab/libsse_head.so 2>&1 | tail -1)" >> $out
  echo "new:  $(timeout 300 python tools/profile_pi.py --atoms 96 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
