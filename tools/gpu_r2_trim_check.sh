#!/bin/bash
# the adaptive Pi operand budget + sse_ctx_trim: Pi tests, the chunk A/B (default now 24 GiB per
# polarity when memory allows), then the full default bench (e2e after trim) at paper scale
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_pi.py tests/test_loop.py -x -q > gpurun_out/r2_trim_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_trim_tests.log
out=gpurun_out/r2_ab_k6chunk2.log; : > $out
for rep in 1 2; do
  echo "chunk 50:  $(SSE_PI_CHUNK_ATOMS=50 timeout 300 python tools/profile_pi.py --atoms 196 --steps 1 2>&1 | tail -1)" >> $out
  echo "default:   $(timeout 300 python tools/profile_pi.py --atoms 196 --steps 1 2>&1 | tail -1)" >> $out
done
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_trim_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_trim_bench.log
