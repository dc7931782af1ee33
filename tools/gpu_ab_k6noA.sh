#!/bin/bash
# K6 diagnostic: the default build vs a measurement-only build whose A operands are register
# constants (tools/ab/libsse_noA.so from a patched copy; wrong results) -> the cost of the G1 gather
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6noA.log; : > $out
for rep in 1 2; do
  echo "default: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "no A:    $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 --lib tools/ab/libsse_noA.so 2>&1 | tail -1)" >> $out
done
cat $out
