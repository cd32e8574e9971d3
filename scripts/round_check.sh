#!/usr/bin/env bash
# Round-end GPU pass: gpu tests, smoke, N=1 bench, reference arm, ncu profile.
set -u
mkdir -p gpurun_out/r01g
nvidia-smi > gpurun_out/r01g/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01g/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01g/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r01g/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r01g/bench_n1.json 2> gpurun_out/r01g/bench_n1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01g/bench_ref.json 2> gpurun_out/r01g/bench_ref.err
timeout 900 bash scripts/profile_round.sh cfg2 r01g
