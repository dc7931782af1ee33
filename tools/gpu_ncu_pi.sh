#!/bin/bash
# Pi kernels: plain timing, then one K6 (default variant) and one K5 launch under ncu --set full
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python tools/profile_pi.py --atoms 96 --steps 1 > gpurun_out/pi_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pi_dmma[34] -s 1 -c 1 -o gpurun_out/pi_k6 -f python tools/profile_pi.py --atoms 96 --steps 1 > gpurun_out/ncu_pi.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pi_build_dmma -s 1 -c 1 -o gpurun_out/pi_k5 -f python tools/profile_pi.py --atoms 96 --steps 1 >> gpurun_out/ncu_pi.log 2>&1
echo "rc=$?"; cat gpurun_out/pi_plain.log
