#!/usr/bin/env bash
# One GPU-box pass: plain bench (the numbers), then the ncu launch list and a
# full capture of the top image-MLP kernels of the SAME command (each ncu pass
# only after the plain run exited 0).  Usage (from the repo root, via gpurun):
#   bash scripts/profile_round.sh <config> <tag>
set -u
CFG=${1:-cfg2}
TAG=${2:-r01}
OUT=gpurun_out/prof_${TAG}_${CFG}
mkdir -p "$OUT"
CMD="python bench.py --config $CFG --steps 4 --warmup 3 --no-e2e --no-cpu-baseline"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/smi.txt" 2>&1
$CMD > "$OUT/plain.log" 2>&1 || { echo "plain run failed"; tail -20 "$OUT/plain.log"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" $CMD > "$OUT/ncu_launches.log" 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:'k_fwd|k_dw0|k_l12|k_dw1|k_sample|k_attn_bwd|k_ref|k_head|k_rows|k_mark' --launch-skip 40 --launch-count 16 \
    -o "$OUT/full" -f $CMD > "$OUT/ncu_full.log" 2>&1
# the layer-0 GEMMs (outside the window above): one launch each, after warm-up
ncu --set full --clock-control none --import-source on -k regex:'k_fwd4|k_dw0p' --launch-skip 4 --launch-count 2 \
    -o "$OUT/gemm" -f $CMD > "$OUT/ncu_gemm.log" 2>&1
echo "done $OUT"
