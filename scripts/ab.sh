#!/bin/bash
# GPU suite, then an alternating A/B of bench.py under two env settings on the
# same box.  Usage: bash scripts/ab.sh <tag> "<envA>" "<envB>" [steps] [skip-tests]
tag=${1:-ab}; A=${2:-X=0}; B=${3:-X=1}; steps=${4:-200}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
if [ -z "$5" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs -x > gpurun_out/${tag}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
fi
for i in 1 2; do
  for e in "$A" "$B"; do
    echo "== $e" >> gpurun_out/${tag}_ab.log
    env $e timeout 600 python bench.py --steps $steps --warmup 5 --no-cpu-baseline --no-e2e >> gpurun_out/${tag}_ab.log 2>&1
  done
done
