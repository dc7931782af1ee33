#!/bin/bash
# K3m at paper (Nkz = Nqz = 3): default KG=2 group + 1-momentum launch vs one KG=3 launch with 2 row
# tiles per warp (SSE_K3M_MT=2); bitwise vs the other K3 kernels first
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k3m_mt2.log; : > $out
timeout 600 python - >> $out 2>&1 <<'PY'
import os, numpy as np
from paper_1912_08810_b200 import inputs, _lib
from paper_1912_08810_b200.types import SimParams, GreensTensor, CombinedD, build_neighbor_map, default_grid
from paper_1912_08810_b200.sse import sse_sigma, SseVariant
import oracle.sse_oracle as orc  # A/B checker only
for (nkz, nqz, ne, nw, na) in [(3, 3, 40, 20, 6), (5, 5, 30, 14, 5), (4, 3, 33, 16, 6)]:
    p = SimParams(n_kz=nkz, n_qz=nqz, n_E=ne, n_w=nw, n_A=na, n_B=4, n_orb=12)
    g_l, g_g, d_l, d_g, dh = inputs.stream_instance(2, p, dh_scale=0.05)
    nmap = build_neighbor_map(p.n_A, p.n_B); grid = default_grid(p)
    dc = CombinedD(*orc.preprocess_D(d_l, d_g, nmap.idx))
    outs = []
    for mt in ("", "2"):
        os.environ["SSE_K3M_MT"] = mt
        o = sse_sigma(SseVariant.BATCHED_FUSED, GreensTensor(g_l, g_g), dc, dh, nmap, grid)
        outs.append((o, _lib.kernel_name("sigma")))
    os.environ["SSE_K3M_MT"] = ""
    eq = np.array_equal(outs[0][0].lesser, outs[1][0].lesser) and np.array_equal(outs[0][0].greater, outs[1][0].greater)
    print(f"Nkz={nkz} Nqz={nqz}: {outs[0][1]} vs {outs[1][1]}: bitwise {eq}")
PY
for rep in 1 2; do
  echo "paper default: $(timeout 300 python tools/profile_sigma.py --atoms 304 --steps 2 2>&1 | tail -1)" >> $out
  echo "paper kg3 mt2: $(SSE_K3M_MT=2 timeout 300 python tools/profile_sigma.py --atoms 304 --steps 2 2>&1 | tail -1)" >> $out
done
cat $out
