#!/bin/bash
# K3 producer-lookahead sweep on a 304-atom paper shard (LAS="..." to choose the values)
export PYTHONUNBUFFERED=1
for LA in ${LAS:-2 4 6 8 11}; do echo "L=$LA $(SSE_SLIDE_LOOKAHEAD=$LA timeout 300 python tools/profile_sigma.py --atoms 304 2>&1 | tail -1)"; done
