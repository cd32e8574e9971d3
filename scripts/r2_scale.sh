#!/bin/bash
# Multi-GPU pass: the multi-GPU parity tests at the box's GPU count, then
# bench lines at N = 1, 2, ..., all GPUs (phase timing on the largest).  Logs: gpurun_out/$1_*
tag=${1:-r2s}
cfg=${2:-cfg2}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
n=$(nvidia-smi -L | wc -l)
if [ -z "$3" ]; then
  timeout 1800 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
fi
for g in 1 2 4 8; do
  [ $g -gt $n ] && break
  if [ $g -eq $n ]; then pt=1; else pt=0; fi
  DICM_PHASE_TIMING=$pt timeout 900 python bench.py --config $cfg --gpus $g --steps 100 --warmup 5 --no-cpu-baseline \
    > gpurun_out/${tag}_${cfg}_n${g}.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_${cfg}_n${g}.log
done
