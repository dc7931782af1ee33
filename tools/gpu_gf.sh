#!/bin/bash
# SURVEY 8f-3 on NCCL: bench at N ranks with the GF-layout phase (two all-to-alls per step)
N=${1:-4}
mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --steps 3 --warmup 3 --cpu-pairs 0 --no-e2e --pi-steps 1 --gf-layout-steps 2 --gf-fused-steps 2 > gpurun_out/bench_gf_n$N.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_gf_n$N.log
tail -3 gpurun_out/bench_gf_n$N.log
