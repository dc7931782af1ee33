#!/bin/bash
# ncu --set full of one K5 launch (the Pi operand build) in the bench (rep < 64 MiB)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
B="bench.py --steps 1 --warmup 1 --no-e2e --cpu-atoms 0 --no-check --phase-device-steps 0"
timeout 600 python $B > gpurun_out/r2_k5_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none -k regex:pi_build_dmma -s 2 -c 1 -o gpurun_out/r2_k5 -f python $B > gpurun_out/r2_ncu_k5.log 2>&1
echo "ncu k5 rc=$?" >> gpurun_out/r2_ncu_k5.log
