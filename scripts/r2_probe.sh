#!/bin/bash
# launch lists of two library builds + a timing A/B with a measurement-only build
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
bash scripts/launches_only.sh cfg2 libhead DICM_LIB_PATH=build/ab/libdicm_b200_HEAD.so
bash scripts/launches_only.sh cfg2 libcur DICM_X=0
DICM_BENCH_NOCHECK=1 bash scripts/abn.sh nostore 100 "DICM_X=0" "DICM_LIB_PATH=build/ab/libdicm_b200_nostore.so"
