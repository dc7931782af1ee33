#!/bin/bash
# K6 v4 split: the whole launch vs the main CTAs alone (tools/ab/libsse_notail.so: tail CTAs exit at
# once; measurement only, wrong results) -> the time the 9th lag tile costs
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6tail.log; : > $out
for rep in 1 2; do
  echo "full:    $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "no tail: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 --lib tools/ab/libsse_notail.so 2>&1 | tail -1)" >> $out
done
cat $out
