export PYTHONUNBUFFERED=1
timeout 200 python -m pytest tests/test_gpu_pi.py -q -m gpu -x 2>&1 | tail -1
timeout 120 python tools/profile_pi.py --atoms 96 --steps 2
