#!/bin/bash
# multi-GPU: the Zipf cluster check + e2e host-timing debug at all GPUs
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
n=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k "zipf or m3n5 or graphs" > gpurun_out/mz_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/mz_pytest.log
DICM_E2E_DEBUG=1 timeout 900 python bench.py --gpus $n --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/mz_bench_n${n}.log 2>&1
