#!/bin/bash
# round-2 evidence pass (current build): smoke, pytest -m gpu, default bench (N=1, all legs), the
# reference arm, small bench, ncu launch list + ncu --set full of one K5 and one K3m (KG=1) launch
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e3_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2e3_smoke.log
timeout 1800 python -m pytest tests -q -m gpu --durations=20 > gpurun_out/r2e3_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2e3_pytest_gpu.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r2e3_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2e3_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2e3_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2e3_bench_ref.log
timeout 600 python bench.py --config small --steps 5 --warmup 3 --no-e2e > gpurun_out/r2e3_bench_small.log 2>&1; echo "rc=$?" >> gpurun_out/r2e3_bench_small.log
B="bench.py --steps 1 --warmup 3 --no-e2e --cpu-atoms 0 --no-check --phase-device-steps 0"
timeout 600 python $B > gpurun_out/r2e3_bench_short.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e3_launches.csv python $B > gpurun_out/r2e3_ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/r2e3_ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pi_build_dmma -s 2 -c 1 -o gpurun_out/r2e3_k5 -f python $B > gpurun_out/r2e3_ncu_k5.log 2>&1
echo "ncu k5 rc=$?" >> gpurun_out/r2e3_ncu_k5.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:kslide -s 5 -c 1 -o gpurun_out/r2e3_k3m_kg1 -f python $B > gpurun_out/r2e3_ncu_k3m_kg1.log 2>&1
echo "ncu k3m kg1 rc=$?" >> gpurun_out/r2e3_ncu_k3m_kg1.log
