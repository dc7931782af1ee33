#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -q -m gpu -k "kheavy or large or multi_gpu" > gpurun_out/pytest_scale.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_scale.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --cpu-pairs 0 > gpurun_out/bench_n2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_n2.log
tail -3 gpurun_out/pytest_scale.log; tail -1 gpurun_out/bench_n2.log
