#!/usr/bin/env bash
# A/B of the k_sample_scatter fork in dicm_sample_bwd (DICM_SAMPLE_FORK=0 = off):
# GPU tests first, then alternating N=1 bench runs on the same box.
set -u
OUT=gpurun_out/ab
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for i in 1 2; do
  DICM_SAMPLE_FORK=0 timeout 600 python bench.py --no-e2e --no-cpu-baseline > $OUT/off_$i.json 2> $OUT/off_$i.err
  timeout 600 python bench.py --no-e2e --no-cpu-baseline > $OUT/on_$i.json 2> $OUT/on_$i.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu.log 2>&1
