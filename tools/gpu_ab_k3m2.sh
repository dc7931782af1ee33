#!/bin/bash
# K3m momentum-group size A/B (SSE_K3M_KG 1/2/3) on paper / small shards + ncu of K3m<12,3>
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
out=gpurun_out/r2_ab_k3m2.log; : > $out
for rep in 1 2; do
  for kg in 1 2 3; do
    echo "paper kg $kg: $(SSE_K3M_KG=$kg timeout 300 python tools/profile_sigma.py --atoms 304 --steps 2 2>&1 | tail -1)" >> $out
    echo "small kg $kg: $(SSE_K3M_KG=$kg timeout 300 python tools/profile_sigma.py --config small --atoms 256 --steps 3 2>&1 | tail -1)" >> $out
  done
done
C="tools/profile_sigma.py --atoms 152 --steps 1"
timeout 300 python $C > gpurun_out/r2_k3m_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:kslide -s 1 -c 1 -o gpurun_out/r2_k3m_paper -f python $C > gpurun_out/r2_ncu_k3m.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2_ncu_k3m.log
cat $out
