#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bench_shapes.py tests/test_gpu_tensorcore.py tests/test_gpu_step.py -x -q > gpurun_out/epi3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/epi3_pytest.log
ABN_ARGS="--config cfg4" bash scripts/abn.sh epi3c4 100 "DICM_FWD4_EPI=1" "DICM_X=0"
bash scripts/abn.sh epi3 200 "DICM_FWD4_EPI=1" "DICM_X=0"
