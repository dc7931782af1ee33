#!/bin/bash
# K3m grouping on kheavy (Nkz=7) and large (Nkz=5) shards: default (KG=2 groups + 1) vs KG=3 with 2
# row tiles per warp (SSE_K3M_MT=2: 3+3+1 / 3+2)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k3m_mt2b.log; : > $out
for rep in 1 2; do
  for cfg in kheavy large; do
    echo "$cfg default: $(timeout 600 python tools/profile_sigma.py --config $cfg --atoms 128 --steps 2 2>&1 | tail -1)" >> $out
    echo "$cfg kg3 mt2: $(SSE_K3M_MT=2 timeout 600 python tools/profile_sigma.py --config $cfg --atoms 128 --steps 2 2>&1 | tail -1)" >> $out
  done
done
cat $out
