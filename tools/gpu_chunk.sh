#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for C in 4 16 48 0; do
  if [ $C -gt 0 ]; then export SSE_OP_CHUNK_ATOMS=$C; else unset SSE_OP_CHUNK_ATOMS; fi
  echo "chunk=$C"; timeout 300 python tools/profile_sigma.py --atoms 148 2>&1 | tail -1
done
