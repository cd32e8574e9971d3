#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_prerank.py -x -q > gpurun_out/hd_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/hd_pytest.log
bash scripts/launches_only.sh cfg2 hdnew DICM_X=0
bash scripts/launches_only.sh cfg2 hdold DICM_LIB_PATH=build/ab/libdicm_b200_HEAD~1.so
