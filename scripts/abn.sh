#!/bin/bash
# Alternating bench A/B/... on one box: bash scripts/abn.sh <tag> <steps> "<envA>" "<envB>" ...
# (optional GPU tests first via ABN_TESTS="tests/x.py ...").  Log: gpurun_out/<tag>_ab.log
tag=$1; steps=$2; shift 2
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
if [ -n "$ABN_TESTS" ]; then
  timeout 1500 python -m pytest $ABN_TESTS -x -q -m gpu > gpurun_out/${tag}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
fi
for i in 1 2 3; do
  for e in "$@"; do
    echo "== $e" >> gpurun_out/${tag}_ab.log
    env $e timeout 600 python bench.py --steps $steps --warmup 5 --no-cpu-baseline --no-e2e ${ABN_ARGS} >> gpurun_out/${tag}_ab.log 2>&1
  done
done
