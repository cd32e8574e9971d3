#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bench_shapes.py -q -k "epilogue" > gpurun_out/misc_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/misc_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/misc_ref2.log 2>&1; echo "rc=$?" >> gpurun_out/misc_ref2.log
timeout 900 python bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/misc_ref2b.log 2>&1; echo "rc=$?" >> gpurun_out/misc_ref2b.log
