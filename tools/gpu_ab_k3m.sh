#!/bin/bash
# K3 single-momentum sliding window (SSE_SIGMA_KERNEL=3) vs multi-momentum (4, default): parity + A/B
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "kernels_bitwise or kernel_shapes or golden or criterion5 or kat or staging or device_api" > gpurun_out/r2_k3m_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k3m_tests.log
out=gpurun_out/r2_ab_k3m.log; : > $out
for rep in 1 2; do
  for c in 3 4; do
    echo "paper kernel $c: $(SSE_SIGMA_KERNEL=$c timeout 300 python tools/profile_sigma.py --atoms 304 --steps 2 2>&1 | tail -1)" >> $out
    echo "small kernel $c: $(SSE_SIGMA_KERNEL=$c timeout 300 python tools/profile_sigma.py --config small --atoms 256 --steps 3 2>&1 | tail -1)" >> $out
  done
done
cat $out
