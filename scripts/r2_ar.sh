#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for i in 1 2; do
for e in "DICM_ALLREDUCE=p2p" "DICM_ALLREDUCE=nccl"; do
  echo "== $e" >> gpurun_out/ar_ab.log
  env $e timeout 900 python bench.py --gpus 4 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e >> gpurun_out/ar_ab.log 2>&1
done; done
