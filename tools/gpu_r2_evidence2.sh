#!/bin/bash
# round-2 evidence after K3m: smoke, full GPU suite, small bench, paper launch list + ncu of one K3m launch
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke3.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke3.log
timeout 1800 python -m pytest tests -q -m gpu --durations=20 > gpurun_out/r2_pytest_gpu3.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu3.log
timeout 600 python bench.py --config small --steps 5 --warmup 3 --no-e2e > gpurun_out/r2_bench_small3.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench_small3.log
B="bench.py --steps 1 --warmup 3 --no-e2e --cpu-atoms 0 --no-check --phase-device-steps 0"
timeout 600 python $B > gpurun_out/r2_bench_short2.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches2.csv python $B > gpurun_out/r2_ncu_launch2.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/r2_ncu_launch2.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:kslide -s 4 -c 1 -o gpurun_out/r2_k3m_bench -f python $B > gpurun_out/r2_ncu_k3m_bench.log 2>&1
echo "ncu k3m rc=$?" >> gpurun_out/r2_ncu_k3m_bench.log
out=gpurun_out/r2_ab_k3m_nw8.log; : > $out
for rep in 1 2; do
  echo "paper 12w kg2 (default): $(timeout 300 python tools/profile_sigma.py --atoms 304 --steps 2 2>&1 | tail -1)" >> $out
  echo "paper 8w kg3: $(SSE_K3M_NW=8 SSE_K3M_KG=3 timeout 300 python tools/profile_sigma.py --atoms 304 --steps 2 2>&1 | tail -1)" >> $out
done
