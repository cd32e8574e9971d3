"""Multi-GPU AMS parity (needs >= 2 GPUs; skipped otherwise): the cluster
against the single-process oracle on the union batch (scripts/cluster_check.py),
with the peer-memory exchange (eager and CUDA-graph steps) and with the NCCL
all-to-all-v exchange; uneven logical topologies (workers != servers != GPUs),
empty local slices, full (unsharded) source models with collect_into_model,
and a DCK1 checkpoint of a sharded run resumed on one GPU."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(world, args, env=None, port=29531):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "scripts", "cluster_check.py")]
    r = subprocess.run(cmd + args, capture_output=True, text=True, timeout=600, env=env)
    if r.returncode:
        print(r.stdout[-6000:])
        print(r.stderr[-6000:])
    assert r.returncode == 0
    return r


def _world():
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    return 4 if n >= 4 else 2


@pytest.mark.parametrize("kind,precision,mode", [("multiquery-attn", "fp32", "eager"), ("sum", "tf32", "eager"),
                                                 ("attn", "bf16", "eager"), ("multiquery-attn", "fp32", "graphs"),
                                                 ("prerank", "fp32", "eager"), ("attn", "fp32", "nccl"),
                                                 ("multiquery-attn", "bf16", "nccl")])
def test_cluster_matches_oracle_on_union(kind, precision, mode):
    world = _world()
    # mode "nccl": the sparse exchanges as NCCL all-to-all-v (DICM_EXCHANGE=nccl)
    # instead of the peer-memory copies, eager steps
    env = dict(os.environ, DICM_EXCHANGE="nccl") if mode == "nccl" else None
    _run(world, [kind, precision, "eager" if mode == "nccl" else mode], env)


@pytest.mark.parametrize("extra", [["--workers", "3", "--servers", "5"], ["--workers", "8", "--servers", "1"],
                                   ["--full-model"], ["--short-last"], ["--workers", "1", "--servers", "3"],
                                   ["--zipf", "1.1"]],
                         ids=["m3n5", "m8n1", "full-model", "short-last", "m1n3", "zipf-hot-keys"])
def test_cluster_topologies_match_oracle(extra):
    """Logical workers / servers mapped onto the GPUs (reference
    tests/test_runtime.py:46-59 runs M = 4, N = 2): results equal the
    oracle on the union batch whatever the topology, including GPUs that
    host no worker (M < G) or get an empty slice of a short union."""
    _run(_world(), ["multiquery-attn", "fp32", "eager"] + extra)


def test_sharded_checkpoint_resumes_on_one_gpu(tmp_path):
    """A multi-GPU run checkpointed through DCK1 (Cluster.collect_into_model
    + Cluster.optimizer_tensors, reference runtime.py:490-516) resumes on a
    single GPU (LocalTrainer + load_warmup) with the same next-iteration loss
    as the cluster's own next iteration."""
    from paper_1711_06505_b200 import checkpoint as CK
    from paper_1711_06505_b200.batch import Batch
    from paper_1711_06505_b200.model import DicmModel
    from paper_1711_06505_b200.pool import FixedExtractor, ImagePool
    from paper_1711_06505_b200.schema import AggregatorSpec, default_schema
    from paper_1711_06505_b200.training import LocalTrainer, TrainConfig
    world = _world()
    path = str(tmp_path / "cluster.dck")
    _run(world, ["multiquery-attn", "fp32", "eager", "--ckpt", path])
    z = np.load(path + ".npz")
    schema = default_schema(3001, 4, 2999, 8, 2000, b_max=30)
    model = DicmModel(schema, AggregatorSpec("multiquery-attn"), None, seed=123)  # values come from the file
    lat = torch.randn((2000, 32), generator=torch.Generator().manual_seed(11))
    pool = ImagePool.from_latents(lat, FixedExtractor(0x5EED, 32, 4096))
    tr = LocalTrainer(model, pool, TrainConfig(batch_size=int(z["size"])))
    ck = CK.load(path)
    assert int(ck.meta["world"]) == world
    CK.load_warmup(ck, model, CK.WarmupMask.full(), fresh_seed=0, trainer=tr)
    onehot = {k[3:]: z[k] for k in z.files if k.startswith("oh/")}
    multi = {k[3:-5]: (z[k], z[k[:-5] + "/off"]) for k in z.files if k.startswith("mh/") and k.endswith("/flat")}
    b = Batch(int(z["size"]), z["labels"], onehot, multi, z["ad"], z["beh"], z["beh_off"])
    loss = tr.train_batch(b)
    assert abs(loss - float(z["loss"])) / max(1.0, abs(loss)) < 1e-5, (loss, float(z["loss"]))
