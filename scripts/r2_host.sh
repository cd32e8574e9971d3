#!/bin/bash
# GPU tests touching the step + e2e host timing at N=1 and all GPUs
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
n=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests/test_gpu_step.py tests/test_gpu_input_pipeline.py tests/test_gpu_multi.py -x -q > gpurun_out/hs_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/hs_pytest.log
DICM_E2E_DEBUG=1 timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/hs_bench_n1.log 2>&1
DICM_E2E_DEBUG=1 timeout 900 python bench.py --gpus $n --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/hs_bench_n${n}.log 2>&1
