#!/usr/bin/env bash
# Round-end pass on 2 GPUs: all GPU tests (incl. multi-GPU), smoke, the N=1
# and N=2 bench lines, and the reference arm.
set -u
OUT=gpurun_out/final
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 \
  bench.py --gpus 2 --steps 200 --warmup 3 > $OUT/bench_n2.json 2> $OUT/bench_n2.err
