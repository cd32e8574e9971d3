#!/bin/bash
# Round-2 GPU check: full GPU suite, smoke, bench (both arms).  Logs in gpurun_out/$1_*.
tag=${1:-r2}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 -rs > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${tag}_bench.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${tag}_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/${tag}_ref.log
