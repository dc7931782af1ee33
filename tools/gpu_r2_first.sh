#!/bin/bash
# round-2 first pass: smoke, GPU tests (incl. the slide goldens, kheavy / large shards), default bench
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/r2_box.txt
free -g >> gpurun_out/r2_box.txt; nproc >> gpurun_out/r2_box.txt; lscpu | head -20 >> gpurun_out/r2_box.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/r2_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench.log
