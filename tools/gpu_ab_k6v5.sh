#!/bin/bash
# K6 v5 (3 warps x 3 lag tiles, no tail CTAs) vs v4 split; Pi parity (incl. the paper-shape golden under v5)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_pi.py -x -q > gpurun_out/r2_k6v5_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k6v5_tests.log
SSE_PI_KERNEL=5 timeout 900 python -m pytest tests/test_gpu_pi.py -x -q -k "golden" > gpurun_out/r2_k6v5_golden.log 2>&1
echo "pytest v5 golden rc=$?" >> gpurun_out/r2_k6v5_golden.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multi_momentum" > gpurun_out/r2_mm_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_mm_tests.log
out=gpurun_out/r2_ab_k6v5.log; : > $out
for rep in 1 2; do
  for v in 4 5; do
    echo "v$v: $(SSE_PI_KERNEL=$v timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  done
done
cat $out
