#!/bin/bash
# Round-end pass on one multi-GPU box: the full GPU suite, smoke, the default
# bench line and its reference arm, cfg2 at N = 2 and 4, cfg1 (both arms),
# cfg3/4/5 at all GPUs.  Logs: gpurun_out/$1_*
tag=${1:-fin}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
n=$(nvidia-smi -L | wc -l)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${tag}_gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 -rs > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 600 python bench.py > gpurun_out/${tag}_cfg2_n1.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_cfg2_n1.log
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_cfg2_ref.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_cfg2_ref.log
for g in 2 4 8; do
  [ $g -gt $n ] && break
  timeout 900 python bench.py --gpus $g --no-cpu-baseline > gpurun_out/${tag}_cfg2_n${g}.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_cfg2_n${g}.log
done
timeout 600 python bench.py --config cfg1 > gpurun_out/${tag}_cfg1_n1.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_cfg1_n1.log
timeout 900 python bench.py --config cfg1 --impl reference > gpurun_out/${tag}_cfg1_ref.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_cfg1_ref.log
for c in cfg3 cfg4 cfg5; do
  timeout 1200 python bench.py --config $c --gpus $n --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_${c}_n${n}.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_${c}_n${n}.log
done
