#!/bin/bash
# K5 W-group size A/B (SSE_PI_WG 9 = round-1 order, 3 default, 1)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k5wg.log; : > $out
for rep in 1 2; do
  for wg in 9 3 1; do
    echo "wg $wg: $(SSE_PI_WG=$wg timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  done
done
cat $out
