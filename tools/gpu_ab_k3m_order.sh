#!/bin/bash
# K3m grid order: row CTAs fastest (SSE_K3_OPTS=3, the previous default) vs the partial row CTAs after
# all full ones (k3_opts bit 2, default 7); Sigma parity tests under the new default first
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k3m_order.log; : > $out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or kernels_bitwise or kernel_shapes or multi_momentum or small_config or paper_config" > gpurun_out/r2_k3m_order_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k3m_order_tests.log
for rep in 1 2; do
  echo "rc fastest: $(SSE_K3_OPTS=3 timeout 300 python tools/profile_sigma.py --atoms 304 --steps 2 2>&1 | tail -1)" >> $out
  echo "tails last: $(timeout 300 python tools/profile_sigma.py --atoms 304 --steps 2 2>&1 | tail -1)" >> $out
  echo "small rc fastest: $(SSE_K3_OPTS=3 timeout 300 python tools/profile_sigma.py --config small --atoms 256 --steps 3 2>&1 | tail -1)" >> $out
  echo "small tails last: $(timeout 300 python tools/profile_sigma.py --config small --atoms 256 --steps 3 2>&1 | tail -1)" >> $out
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --cpu-atoms 0 --pi-steps 0 --phase-device-steps 0 > gpurun_out/r2_k3m_order_bench.log 2>&1
SSE_K3_OPTS=3 timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --cpu-atoms 0 --pi-steps 0 --phase-device-steps 0 > gpurun_out/r2_k3m_order_bench_old.log 2>&1
cat $out
