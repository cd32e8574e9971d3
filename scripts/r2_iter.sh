#!/bin/bash
# one iteration: the GPU tests given in $2 (default: all), then a cfg2 launch list + bench
tag=${1:-it}; tests=${2:-tests}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest $tests -x -q -m gpu > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
bash scripts/launches_only.sh cfg2 $tag DICM_X=0
