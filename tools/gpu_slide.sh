#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for K in ${KS:-4 3}; do echo "K=$K"; SSE_SIGMA_KERNEL=$K timeout 300 python tools/profile_sigma.py --atoms 148 2>&1 | tail -1; done
for K in ${TK:-4}; do SSE_SIGMA_KERNEL=$K timeout 900 python -m pytest tests -x -q -m gpu -k "not paper_config" 2>&1 | tail -1; done
