#!/bin/bash
# K6 (Pi chains) ncu capture: plain run first, then one launch under ncu --set full
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 120 python -m pytest tests/test_gpu_pi.py -q -m gpu -x 2>&1 | tail -2
timeout 120 python tools/profile_pi.py --atoms 96 --steps 1 > gpurun_out/pi_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pi_dmma -s 1 -c 1 -o gpurun_out/pi_k6v2 -f python tools/profile_pi.py --atoms 96 --steps 1 > gpurun_out/ncu_pi.log 2>&1
echo "rc=$?"; cat gpurun_out/pi_plain.log
