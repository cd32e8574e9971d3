#!/usr/bin/env bash
# cfg3/cfg4/cfg5 bench lines at N=4 (run under gpurun --gpus 4).
set -u
OUT=gpurun_out/cfgs
mkdir -p $OUT
for C in cfg3 cfg4 cfg5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 4 --config $C --steps 50 --warmup 10 > $OUT/bench_${C}_n4.json 2> $OUT/bench_${C}_n4.err
done
