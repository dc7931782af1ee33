#!/bin/bash
# evidence refresh after a K3 change: smoke, fused SSE phase bench, ncu launch list, ncu --set full of one K3 launch
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 1 --warmup 3 --no-e2e --cpu-pairs 0 --pi-steps 0 --phase-steps 2 > gpurun_out/bench_phase.log 2>&1; echo "bench phase rc=$?" >> gpurun_out/bench_phase.log
B="bench.py --steps 1 --warmup 3 --no-e2e --cpu-pairs 0 --no-check"
timeout 600 python $B > gpurun_out/bench_short.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python $B > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sigma_dmma -s 4 -c 1 -o gpurun_out/bench_k3 -f python $B > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/bench_phase.log; tail -1 gpurun_out/ncu_launch.log; tail -1 gpurun_out/ncu_full.log
