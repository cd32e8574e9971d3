#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
DICM_FWD4_EPI=2 timeout 900 python -m pytest tests/test_gpu_bench_shapes.py tests/test_gpu_tensorcore.py -x -q > gpurun_out/epi_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/epi_pytest.log
DICM_BENCH_NOCHECK=1 bash scripts/abn.sh epi 200 "DICM_FWD4_EPI=1" "DICM_FWD4_EPI=2" "DICM_LIB_PATH=build/ab/libdicm_b200_nostore.so"
