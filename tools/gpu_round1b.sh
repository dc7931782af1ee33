#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-pairs 2 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python tools/profile_sigma.py > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sigma_dmma -s 1 -c 1 -o gpurun_out/sigma_full -f python tools/profile_sigma.py > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --cpu-pairs 0 --no-check > gpurun_out/bench_short.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --cpu-pairs 0 --no-check > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
tail -3 gpurun_out/bench.log; cat gpurun_out/prof_plain.log; tail -3 gpurun_out/ncu_full.log; tail -3 gpurun_out/ncu_launch.log
