#!/bin/bash
# full single-GPU evidence pass: tests, smoke, bench, ncu launch list, ncu full captures of K3 (bench),
# K6 and K5 (Pi, 98-atom paper shard), the fused SSE phase from host memory
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --steps 1 --warmup 3 --no-e2e --cpu-pairs 0 --pi-steps 0 --phase-steps 2 > gpurun_out/bench_phase.log 2>&1; echo "bench phase rc=$?" >> gpurun_out/bench_phase.log
B="bench.py --steps 1 --warmup 3 --no-e2e --cpu-pairs 0 --no-check"
timeout 600 python $B > gpurun_out/bench_short.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python $B > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sigma_dmma -s 4 -c 1 -o gpurun_out/bench_k3 -f python $B > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
timeout 300 python tools/profile_pi.py --atoms 96 --steps 1 > gpurun_out/pi_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pi_dmma[34] -s 1 -c 1 -o gpurun_out/pi_k6 -f python tools/profile_pi.py --atoms 96 --steps 1 > gpurun_out/ncu_pi.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pi_build_dmma -s 1 -c 1 -o gpurun_out/pi_k5 -f python tools/profile_pi.py --atoms 96 --steps 1 >> gpurun_out/ncu_pi.log 2>&1
echo "ncu pi rc=$?" >> gpurun_out/ncu_pi.log
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/bench.log; tail -1 gpurun_out/bench_phase.log; tail -1 gpurun_out/ncu_launch.log; tail -1 gpurun_out/ncu_full.log; tail -1 gpurun_out/ncu_pi.log; cat gpurun_out/pi_plain.log
