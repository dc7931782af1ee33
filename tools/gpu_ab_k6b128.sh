#!/bin/bash
# K6 v4 split: B pairs by two LDS.64 (default) vs one LDS.128 + selects, per-n-tile x/y order
# (SSE_PI_B128=1); bitwise check of the Pi tests under the switch first
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6b128.log; : > $out
SSE_PI_B128=1 timeout 900 python -m pytest tests/test_gpu_pi.py -x -q -k "split or shapes" > gpurun_out/r2_k6b128_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k6b128_tests.log
timeout 300 python - >> $out 2>&1 <<'PY'
import os, numpy as np
from paper_1912_08810_b200 import inputs, _lib
from paper_1912_08810_b200.types import SimParams, GreensTensor, build_neighbor_map, default_grid
from paper_1912_08810_b200.sse import sse_pi
p = SimParams(n_kz=3, n_qz=3, n_E=50, n_w=70, n_A=5, n_B=4, n_orb=12)
g_l, g_g, _, _, dh = inputs.stream_instance(4, p, dh_scale=0.05)
nmap = build_neighbor_map(p.n_A, p.n_B); grid = default_grid(p)
outs = []
for b in ("", "1"):
    os.environ["SSE_PI_B128"] = b
    outs.append(sse_pi(GreensTensor(g_l, g_g), dh, nmap, grid, p.n_qz))
print("paper-shaped Pi, B128 vs default bitwise:", np.array_equal(outs[0].lesser, outs[1].lesser) and np.array_equal(outs[0].greater, outs[1].greater))
PY
for rep in 1 2; do
  echo "lds64:  $(timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
  echo "lds128: $(SSE_PI_B128=1 timeout 300 python tools/profile_pi.py --atoms 98 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
