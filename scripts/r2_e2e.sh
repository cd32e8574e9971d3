#!/bin/bash
# GPU suite + bench with both e2e APIs (host pipeline A/B).  Logs: gpurun_out/$1_*
tag=${1:-r2e}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
for api in stream batch stream batch; do
  DICM_E2E_DEBUG=1 DICM_E2E_API=$api timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline >> gpurun_out/${tag}_bench_${api}.log 2>&1
done
