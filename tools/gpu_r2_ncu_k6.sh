#!/bin/bash
# ncu --set full (with source) of one K6 launch (Pi chains, 4-slot v4 split) on a 96-atom Pi
# chunk: stall reasons per SASS line for the next K6 step (rep < 64 MiB)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
timeout 300 python tools/profile_pi.py --atoms 96 --steps 1 > gpurun_out/r2_k6_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pi_dmma4 -s 1 -c 1 \
    -o gpurun_out/r2_k6${TAG} -f python tools/profile_pi.py --atoms 96 --steps 1 > gpurun_out/r2_ncu_k6.log 2>&1
echo "ncu k6 rc=$?" >> gpurun_out/r2_ncu_k6.log
