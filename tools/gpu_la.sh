#!/bin/bash
export PYTHONUNBUFFERED=1
for LA in 2 4 6 8 11; do echo "L=$LA"; SSE_SLIDE_LOOKAHEAD=$LA timeout 300 python tools/profile_sigma.py --atoms 148 2>&1 | tail -1; done
