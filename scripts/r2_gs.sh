#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
n=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/gs_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gs_pytest.log
timeout 900 python bench.py --gpus $n --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/gs_n${n}.log 2>&1
timeout 900 python bench.py --gpus 2 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/gs_n2.log 2>&1
