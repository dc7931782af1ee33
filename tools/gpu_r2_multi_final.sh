#!/bin/bash
# final build on N GPUs (gpurun --gpus N): host memory / cores, the multi-GPU tests, and the default
# bench under torchrun exactly as the driver launches it (plus the GF-layout legs)
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
N=$(nvidia-smi -L | wc -l)
{ free -g; nproc; nvidia-smi topo -m | head -12; } > gpurun_out/r2f_host_n$N.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scatter.py -q -k "in_library_multi or peer_scatter or multi_gpu" > gpurun_out/r2f_multi_tests_n$N.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2f_multi_tests_n$N.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/r2f_bench_n$N.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2f_bench_n$N.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus $N --steps 2 --warmup 3 --no-e2e --cpu-atoms 0 --pi-steps 0 --phase-device-steps 0 \
  --gf-fused-steps 1 --gf-layout-steps 1 > gpurun_out/r2f_bench_gf_n$N.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2f_bench_gf_n$N.log
