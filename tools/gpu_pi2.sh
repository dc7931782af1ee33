export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_pi.py -q -m gpu -x 2>&1 | tail -3
for k in 1 2; do echo "SSE_PI_KERNEL=$k"; SSE_PI_KERNEL=$k timeout 300 python tools/profile_pi.py --atoms 148; done
