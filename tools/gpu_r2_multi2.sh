#!/bin/bash
# multi-GPU: in-library NCCL path test, e2e with the per-rank host thread share
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scatter.py -q -k "in_library_multi or peer_scatter or multi_gpu" > gpurun_out/r2_multi2_tests_n$N.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_multi2_tests_n$N.log
SSE_STAGING_TRACE=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 3 --warmup 3 --pi-steps 0 --phase-device-steps 0 > gpurun_out/r2_bench2_n$N.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench2_n$N.log
