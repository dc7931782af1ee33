#!/bin/bash
# N = 4: multi-GPU tests + the default bench under torchrun (driver's launch) + ncu capture of the K3m KG=1 launch on GPU 0 is NOT done here
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scatter.py -q -k "in_library_multi or peer_scatter or multi_gpu" > gpurun_out/r2_multi_tests_n$N.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_multi_tests_n$N.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 5 --warmup 3 --gf-fused-steps 1 --gf-layout-steps 1 > gpurun_out/r2_bench_n$N.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench_n$N.log
