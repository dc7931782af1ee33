#!/bin/bash
# kheavy (Nkz = Nqz = 7) and large (NA = 10240, NE = 1220, Nkz = Nqz = 5) under torchrun on the box's GPUs
cd "$GRAFT_REPO_ROOT"
export PYTHONUNBUFFERED=1
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --config kheavy --gpus $N --steps 3 --warmup 3 --no-e2e --phase-device-steps 0 > gpurun_out/r2f_bench_kheavy_n$N.log 2>&1
echo "rc=$?" >> gpurun_out/r2f_bench_kheavy_n$N.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --config large --gpus $N --steps 2 --warmup 3 --no-e2e --pi-steps 0 --phase-device-steps 0 > gpurun_out/r2f_bench_large_n$N.log 2>&1
echo "rc=$?" >> gpurun_out/r2f_bench_large_n$N.log
