"""Multi-GPU AMS parity (needs >= 2 GPUs; skipped otherwise): the cluster
against the single-process oracle on the union batch (scripts/cluster_check.py),
with the peer-memory exchange (eager and CUDA-graph steps) and with the NCCL
all-to-all-v exchange."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("kind,precision,mode", [("multiquery-attn", "fp32", "eager"), ("sum", "tf32", "eager"),
                                                 ("attn", "bf16", "eager"), ("multiquery-attn", "fp32", "graphs"),
                                                 ("prerank", "fp32", "eager"), ("attn", "fp32", "nccl"),
                                                 ("multiquery-attn", "bf16", "nccl")])
def test_cluster_matches_oracle_on_union(kind, precision, mode):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = 4 if n >= 4 else 2
    # mode "nccl": the sparse exchanges as NCCL all-to-all-v (DICM_EXCHANGE=nccl)
    # instead of the peer-memory copies, eager steps
    env = dict(os.environ, DICM_EXCHANGE="nccl") if mode == "nccl" else None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29531", os.path.join(ROOT, "scripts", "cluster_check.py"),
           kind, precision, "eager" if mode == "nccl" else mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
