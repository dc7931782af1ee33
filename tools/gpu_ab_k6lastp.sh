#!/bin/bash
# K6 v4 split at 3 CTAs / SM: fixed producer warp vs last-releaser refill (LASTP), 4 and 5 slots
# (the LASTP variant and SSE_PI_V4_LASTP were removed after this A/B: no difference, `profiles/r02_ab_k6_lastp_rejected.log`)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6lastp.log; : > $out
SSE_PI_V4_MINB=3 SSE_PI_V4_LASTP=1 timeout 600 python -m pytest tests/test_gpu_pi.py -x -q -k "split" > gpurun_out/r2_k6lastp_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k6lastp_tests.log
export SSE_PI_V4_MINB=3
for rep in 1 2; do
  echo "minb3 4 slots:       $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "minb3 4 slots lastp: $(SSE_PI_V4_LASTP=1 timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "minb3 5 slots lastp: $(SSE_PI_V4_LASTP=1 SSE_PI_V4_SLOTS=5 timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
