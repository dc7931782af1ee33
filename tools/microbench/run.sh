#!/bin/bash
# host facts + FP64 peak microbenchmark on the GPU box
mkdir -p gpurun_out
{ nproc; free -g; lscpu | head -20; nvidia-smi; } > gpurun_out/host_info.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/fp64_clocks.csv &
SMI=$!
./tools/microbench/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
kill $SMI
cat gpurun_out/fp64_peak.txt
