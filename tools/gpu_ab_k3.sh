#!/bin/bash
# A/B of the sliding-window K3 options on a 304-atom paper shard (HEAD build vs SSE_K3_OPTS 0..3)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
out=gpurun_out/ab_k3.log; : > $out
for rep in 1 2; do
  echo "head: $(timeout 300 python tools/profile_sigma.py --atoms 304 --steps 2 --lib tools/ab/libsse_head.so 2>&1 | tail -1)" >> $out
  for o in ${OPTS:-0 1 2 3}; do
    echo "opts $o: $(SSE_K3_OPTS=$o timeout 300 python tools/profile_sigma.py --atoms 304 --steps 2 2>&1 | tail -1)" >> $out
  done
done
cat $out
