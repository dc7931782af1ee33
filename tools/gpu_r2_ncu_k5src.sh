#!/bin/bash
# ncu --set full (with source) of one K5 launch (Pi operand build) on a 96-atom paper Pi chunk
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
timeout 300 python tools/profile_pi.py --atoms 96 --steps 1 > gpurun_out/r2_k5_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pi_build_dmma -s 1 -c 1 \
    -o gpurun_out/r2_k5src -f python tools/profile_pi.py --atoms 96 --steps 1 > gpurun_out/r2_ncu_k5src.log 2>&1
echo "ncu k5 rc=$?" >> gpurun_out/r2_ncu_k5src.log
