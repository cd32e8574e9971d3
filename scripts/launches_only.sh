#!/usr/bin/env bash
# Plain bench of one config at N=1, then its ncu launch list (same command).
#   bash scripts/launches_only.sh <config> <tag> [extra env assignments...]
set -u
CFG=${1:-cfg2}; TAG=${2:-x}; shift 2 || true
OUT=gpurun_out/launch_${TAG}_${CFG}
mkdir -p "$OUT"
CMD="python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline"
env "$@" $CMD > "$OUT/plain.log" 2>&1 || { echo "plain run failed"; tail -20 "$OUT/plain.log"; exit 1; }
env "$@" ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" python bench.py --config $CFG --steps 4 --warmup 3 --no-e2e --no-cpu-baseline \
    > "$OUT/ncu_launches.log" 2>&1
echo "done $OUT"
