#!/bin/bash
# K6 launch size: the same 100-atom paper Pi as 2 launches of 50 atoms (default VT budget) vs one of 100
# (SSE_PI_CHUNK_ATOMS=100) vs 4 of 25 -> how much the per-launch drain costs
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6chunk.log; : > $out
for rep in 1 2; do
  echo "chunk 50 (default): $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "chunk 100:          $(SSE_PI_CHUNK_ATOMS=100 timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "chunk 25:           $(SSE_PI_CHUNK_ATOMS=25 timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
