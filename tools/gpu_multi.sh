#!/bin/bash
# multi-GPU pass: N-GPU parity tests + torchrun bench at N ranks
N=${1:-2}
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -x -q -m gpu -k "multi_gpu or paper_config or kheavy or large" > gpurun_out/pytest_multi_$N.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_multi_$N.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 3 --warmup 3 --cpu-pairs 0 > gpurun_out/bench_n$N.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_n$N.log
tail -4 gpurun_out/pytest_multi_$N.log; tail -4 gpurun_out/bench_n$N.log
