"""The multi-GPU step's host-side exchange logic on CPU (gloo, world size 2):
count exchange, all-to-all-v of keys / rows and the owner-side ordering the
device kernels rely on (requests sorted per owner, responses in request
order, pushes grouped by source in ascending rank order)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bucket(keys, world):
    """numpy restatement of dicm_bucket_by_owner: stable partition by owner."""
    owner = keys % world
    order = np.argsort(owner, kind="stable")
    send = (keys[order] // world).astype(np.int32)
    counts = np.bincount(owner, minlength=world).astype(np.int32)
    perm = np.empty(len(keys), dtype=np.int64)
    perm[order] = np.arange(len(keys))
    return send, counts, perm


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_06505_b200.runtime import _a2a, exchange_counts
        rng = np.random.default_rng(rank)
        P = 1000
        uniq = np.unique(rng.integers(0, P, 200)).astype(np.int64)      # local dedup output
        send, counts, perm = _bucket(uniq, world)
        pair = torch.tensor(np.stack([counts, counts * 0 + 1], 1), dtype=torch.int32)
        sent, recv = exchange_counts(pair)
        si, ri = sent[:, 0].tolist(), recv[:, 0].tolist()
        rk = torch.empty(sum(ri), dtype=torch.int32)
        _a2a(rk, torch.as_tensor(send), ri, si)
        # owner: every received key is ours; per source the keys stay sorted
        got = rk.numpy()
        off = np.concatenate([[0], np.cumsum(ri)])
        ok = all(np.all(np.diff(got[off[s]:off[s + 1]]) > 0) for s in range(world))
        ok &= bool(np.all(got >= 0)) and bool(np.all(got < (P + world - 1) // world))
        # owner answers row i of its request list with a row derived from the key
        resp = torch.tensor(np.repeat((got * world + rank)[:, None], 12, 1), dtype=torch.float32)
        back = torch.empty((sum(si), 12), dtype=torch.float32)
        _a2a(back, resp, si, ri)
        emb = back.numpy()[perm]            # requester: back to unique order
        ok &= bool(np.array_equal(emb[:, 0], uniq.astype(np.float32)))
        # push rows back to owners grouped by source
        push = torch.tensor(emb[np.argsort(perm)], dtype=torch.float32)
        recv_rows = torch.empty((sum(ri), 12), dtype=torch.float32)
        _a2a(recv_rows, push, ri, si)
        ok &= bool(np.array_equal(recv_rows.numpy()[:, 0], (got * world + rank).astype(np.float32)))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_exchange_roundtrip_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
