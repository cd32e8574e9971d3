#!/bin/bash
# The other BASELINE configs: cfg1 at N=1 (both arms), cfg3/cfg4/cfg5 at all GPUs.  Logs: gpurun_out/$1_*
tag=${1:-r2c}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
n=$(nvidia-smi -L | wc -l)
timeout 600 python bench.py --config cfg1 --steps 100 --warmup 5 > gpurun_out/${tag}_cfg1_n1.log 2>&1
timeout 900 python bench.py --config cfg1 --impl reference --steps 20 --warmup 5 > gpurun_out/${tag}_cfg1_ref.log 2>&1
for c in cfg3 cfg4 cfg5; do
  timeout 1200 python bench.py --config $c --gpus $n --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_${c}_n${n}.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_${c}_n${n}.log
done
