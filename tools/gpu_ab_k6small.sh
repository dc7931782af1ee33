#!/bin/bash
# small config (No=10, Nw=16) K6 q-in-warps: 9-warp CTA at 72 registers (spills) vs 6-warp CTAs
# at 2 / 3 / 4 CTAs per SM; bitwise check of the variants on a small shard, then timing
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k6small.log; : > $out
SSE_PI_QW=3 timeout 600 python -m pytest tests/test_gpu_pi.py -x -q -k "shapes or small" > gpurun_out/r2_k6small_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_k6small_tests.log
timeout 600 python - >> $out 2>&1 <<'PY'
import os, numpy as np
from paper_1912_08810_b200 import inputs, _lib
from paper_1912_08810_b200.types import SimParams, GreensTensor, build_neighbor_map, default_grid
from paper_1912_08810_b200.sse import sse_pi
p = SimParams(n_kz=3, n_qz=3, n_E=64, n_w=16, n_A=9, n_B=4, n_orb=10)
g_l, g_g, _, _, dh = inputs.stream_instance(3, p, dh_scale=0.05)
nmap = build_neighbor_map(p.n_A, p.n_B); grid = default_grid(p)
ref = None
for qw in ("", "2", "3", "4"):
    os.environ["SSE_PI_QW"] = qw
    o = sse_pi(GreensTensor(g_l, g_g), dh, nmap, grid, p.n_qz)
    name = _lib.kernel_name("pi")
    if ref is None: ref = o
    print(f"QW={qw or 'default'}: {name}: bitwise {np.array_equal(o.lesser, ref.lesser) and np.array_equal(o.greater, ref.greater)}")
PY
for rep in 1 2; do
  for qw in "" 2 3 4; do
    echo "QW=${qw:-default}: $(SSE_PI_QW=$qw timeout 300 python tools/profile_pi.py --config small --atoms 256 --steps 2 2>&1 | tail -1)" >> $out
  done
done
cat $out
