#!/bin/bash
# ncu launch list (gpu__time_duration per launch) of the default bench legs that carry the roofline
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
B="bench.py --steps 1 --warmup 3 --no-e2e --cpu-atoms 0 --no-check --phase-device-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_final.csv \
  python $B > gpurun_out/r2_ncu_launches_final.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/r2_ncu_launches_final.log
