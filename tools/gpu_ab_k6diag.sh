#!/bin/bash
# K6 diagnostics (measurement-only builds from patched copies in tools/ab/, wrong results): the
# default build vs A operands as register constants (noA), B operands of the two-tile warps as
# constants (noB), and both (noAB: DMMAs + the real V ring, stage loop and launch structure)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6diag.log; : > $out
for rep in 1 2; do
  echo "default: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  for v in noA noB noAB; do
    echo "$v: $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 --lib tools/ab/libsse_$v.so 2>&1 | tail -1)" >> $out
  done
done
cat $out
