#!/bin/bash
# the odd-Nkz K3m grouping (pairs + one 3-momentum group at 2 row tiles, default) vs the plain pairs +
# 1-momentum remainder (SSE_K3M_MT=3) on paper (3), large (2+3) and kheavy (2+2+3) shards
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k3m_odd.log; : > $out
for rep in 1 2; do
  for cfg in paper large kheavy; do
    a=128; [ $cfg = paper ] && a=304
    echo "$cfg pairs+1:  $(SSE_K3M_MT=3 timeout 600 python tools/profile_sigma.py --config $cfg --atoms $a --steps 2 2>&1 | tail -1)" >> $out
    echo "$cfg pairs+3: $(timeout 600 python tools/profile_sigma.py --config $cfg --atoms $a --steps 2 2>&1 | tail -1)" >> $out
  done
done
cat $out
