#!/bin/bash
# hot-key passes: step tests, then cfg4 and cfg2 benches (logs gpurun_out/$1_*)
tag=${1:-hot}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py --config cfg4 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_cfg4.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_cfg2.log 2>&1
