#!/bin/bash
# round-2 evidence: staging timeline, ncu launch list of the paper bench, ncu --set full of one
# K3 launch at paper (slide<12>) and at small (slide<10>)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
SSE_STAGING_TRACE=1 timeout 900 python bench.py --steps 1 --warmup 3 --cpu-atoms 0 --pi-steps 0 \
  --phase-device-steps 0 --e2e-steps 1 --e2e-warmup 1 > gpurun_out/r2_staging_trace.log 2>&1
echo "trace rc=$?" >> gpurun_out/r2_staging_trace.log
B="bench.py --steps 1 --warmup 3 --no-e2e --cpu-atoms 0 --no-check --phase-device-steps 0"
timeout 600 python $B > gpurun_out/r2_bench_short.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python $B > gpurun_out/r2_ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/r2_ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sigma_dmma_slide -s 4 -c 1 -o gpurun_out/r2_k3_paper -f python $B > gpurun_out/r2_ncu_k3_paper.log 2>&1
echo "ncu k3 paper rc=$?" >> gpurun_out/r2_ncu_k3_paper.log
S="bench.py --config small --steps 1 --warmup 3 --no-e2e --cpu-atoms 0 --no-check --pi-steps 0 --phase-device-steps 0"
timeout 600 python $S > gpurun_out/r2_bench_small_short.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sigma_dmma_slide -s 4 -c 1 -o gpurun_out/r2_k3_small -f python $S > gpurun_out/r2_ncu_k3_small.log 2>&1
echo "ncu k3 small rc=$?" >> gpurun_out/r2_ncu_k3_small.log
