#!/bin/bash
# K3m: combined fragments for No = 10 (parity + A/B vs side-by-side vectors), default kg per No, bench lines
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "kernels_bitwise or kernel_shapes or golden or criterion5 or kat or staging or device_api or small_config" > gpurun_out/r2_k3m3_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k3m3_tests.log
out=gpurun_out/r2_ab_k3m3.log; : > $out
for rep in 1 2; do
  echo "paper default: $(timeout 300 python tools/profile_sigma.py --atoms 304 --steps 2 2>&1 | tail -1)" >> $out
  echo "small comb: $(timeout 300 python tools/profile_sigma.py --config small --atoms 256 --steps 3 2>&1 | tail -1)" >> $out
  echo "small nocomb kg3: $(SSE_K3M_COMB=0 timeout 300 python tools/profile_sigma.py --config small --atoms 256 --steps 3 2>&1 | tail -1)" >> $out
done
timeout 600 python bench.py --config small --steps 5 --warmup 3 --no-e2e > gpurun_out/r2_bench_small2.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench_small2.log
timeout 900 python bench.py --steps 3 --warmup 3 --pi-steps 0 --phase-device-steps 0 > gpurun_out/r2_bench_paper2.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench_paper2.log
cat $out
