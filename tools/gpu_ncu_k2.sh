#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
export SSE_SIGMA_KERNEL=3
timeout 300 python tools/profile_sigma.py > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sigma_dmma -s 1 -c 1 -o gpurun_out/sigma_slide12 -f python tools/profile_sigma.py > gpurun_out/ncu_tma.log 2>&1
echo "rc=$?"
