#!/bin/bash
# full GPU test suite + smoke + small-config bench (No = 10 production K3) + paper Sigma-only bench
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke2.log
timeout 1800 python -m pytest tests -q -m gpu --durations=25 -p no:randomly > gpurun_out/r2_pytest_gpu2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu2.log
timeout 600 python bench.py --config small --steps 5 --warmup 3 --no-e2e --phase-device-steps 1 > gpurun_out/r2_bench_small.log 2>&1
echo "rc=$?" >> gpurun_out/r2_bench_small.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --cpu-atoms 0 --pi-steps 0 --phase-device-steps 0 > gpurun_out/r2_bench_paper_k3.log 2>&1
echo "rc=$?" >> gpurun_out/r2_bench_paper_k3.log
