#!/bin/bash
# Round-2 2/4-GPU pass: the multi-GPU parity tests, then bench lines at N=1 (A/B of one
# env switch if given) and N=world.  Logs in gpurun_out/$1_*.
tag=${1:-r2m}
ab=${2:-}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
n=$(nvidia-smi -L | wc -l)
timeout 1800 python -m pytest tests/test_gpu_multi.py tests/test_gpu_step.py -q -p no:cacheprovider -x > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench_n1.log 2>&1
if [ -n "$ab" ]; then env $ab timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench_n1_ab.log 2>&1; fi
DICM_PHASE_TIMING=1 timeout 600 python bench.py --gpus $n --steps 100 --warmup 5 > gpurun_out/${tag}_bench_n${n}.log 2>&1
echo "bench rc=$?" >> gpurun_out/${tag}_bench_n${n}.log
