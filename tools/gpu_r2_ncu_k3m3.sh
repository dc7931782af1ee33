#!/bin/bash
# ncu --set full of one production K3m launch (<12,12,2,3>: all 3 momenta of a 277-atom operator
# chunk, both polarities) in the paper bench -> roofline traffic (rep < 64 MiB)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
B="bench.py --steps 1 --warmup 3 --no-e2e --cpu-atoms 0 --no-check --phase-device-steps 0 --pi-steps 0"
timeout 600 python $B > gpurun_out/r2_k3m3_plain.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none -k regex:kslide -s 3 -c 1 -o gpurun_out/r2_k3m3 -f python $B > gpurun_out/r2_ncu_k3m3.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2_ncu_k3m3.log
