#!/bin/bash
export PYTHONUNBUFFERED=1
timeout 200 python -m pytest tests/test_gpu_pi.py -q -m gpu -x 2>&1 | tail -2
for pr in 0 1; do echo "SSE_PI_PRODUCER=$pr"; SSE_PI_PRODUCER=$pr timeout 120 python tools/profile_pi.py --atoms 96 --steps 2; done
