#!/usr/bin/env bash
# Multi-GPU pass (run under gpurun --gpus 4): the multi-GPU tests, then the
# N=2 and N=4 bench lines launched the way the driver launches them.
set -u
OUT=gpurun_out/multi
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --gpus $N --steps 200 --warmup 3 > $OUT/bench_n$N.json 2> $OUT/bench_n$N.err
done
