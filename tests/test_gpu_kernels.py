"""Kernel-level parity on the B200: dedup, pool gather/materialize, exchange
helpers.  Integer / byte work is compared bit-exactly."""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_1711_06505_b200 import _lib
    assert torch.cuda.is_available()
    assert _lib.lib.dicm_device_arch() >= 100
    return _lib


def run_dedup(L, arrays, vocabs, bases=None, tag=0):
    dev = "cuda"
    bases = bases or [0] * len(arrays)
    space = max(b + v for b, v in zip(bases, vocabs))
    ts = [torch.as_tensor(np.asarray(a, dtype=np.int32), device=dev) for a in arrays]
    n = sum(len(a) for a in arrays)
    segs, off = [], 0
    for t, b, v in zip(ts, bases, vocabs):
        segs.append(L.KeySeg(t.data_ptr(), t.numel(), b, v, off))
        off += t.numel()
    ws = torch.empty(L.lib.dicm_dedup_workspace(space), dtype=torch.uint8, device=dev)
    uniq = torch.full((max(n, 1),), -7, dtype=torch.int32, device=dev)
    inv = torch.full((max(n, 1),), -7, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    status = torch.zeros(8, dtype=torch.int32, device=dev)
    arr = (L.KeySeg * len(segs))(*segs)
    L.check(L.lib.dicm_dedup(arr, len(segs), space, ws.data_ptr(), ws.numel(), uniq.data_ptr(), inv.data_ptr(),
                             cnt.data_ptr(), tag, status.data_ptr(), L.stream_handle()))
    torch.cuda.synchronize()
    k = int(cnt.item())
    return uniq[:k].cpu().numpy(), inv[:n].cpu().numpy(), status.cpu().numpy()


@pytest.mark.parametrize("dist", ["uniform", "zipf", "dense", "single"])
@pytest.mark.parametrize("n,space", [(1, 1), (1000, 10), (823296, 1_000_000), (200_000, 20_000_000)])
def test_dedup_bitexact_vs_numpy(L, dist, n, space):
    from paper_1711_06505_b200.batch import zipf_keys
    rng = np.random.default_rng(n + space)
    if dist == "uniform":
        keys = rng.integers(0, space, n)
    elif dist == "zipf":
        keys = zipf_keys(rng, n, space, 1.1)
    elif dist == "dense":
        keys = rng.permutation(np.arange(space))[:n] if n <= space else rng.integers(0, space, n)
    else:
        keys = np.full(n, space - 1)
    u, inv, st = run_dedup(L, [keys], [space])
    ref_u = np.unique(keys)
    assert st[0] == 0
    assert np.array_equal(u, ref_u)                      # model.py:187
    assert np.array_equal(inv, np.searchsorted(ref_u, keys))  # model.py:374/378


def test_dedup_multi_segment_key_space(L):
    rng = np.random.default_rng(3)
    vocabs = [100_000, 4, 100_000, 8, 100_000, 1_000_000, 1_000_000]
    bases = list(np.concatenate([[0], np.cumsum(vocabs)[:-1]]))
    arrays = [rng.integers(0, v, 4096 if i < 4 or i == 5 else 50_000) for i, v in enumerate(vocabs)]
    u, inv, st = run_dedup(L, arrays, vocabs, bases)
    keys = np.concatenate([a + b for a, b in zip(arrays, bases)])
    ref_u = np.unique(keys)
    assert np.array_equal(u, ref_u)
    assert np.array_equal(inv, np.searchsorted(ref_u, keys))


def test_dedup_empty_segment_and_oov_flag(L):
    u, inv, st = run_dedup(L, [np.array([], dtype=np.int64), np.array([3, 1, 3])], [10, 10])
    assert np.array_equal(u, [1, 3]) and np.array_equal(inv, [1, 0, 1])
    u, inv, st = run_dedup(L, [np.array([2, 12, 5])], [10], tag=1)
    assert st[0] == 1 and st[1] == 12 and st[2] == 16  # tag 1, segment 0
    assert np.array_equal(u, [2, 5]) and inv[1] == 0     # OOV inverse kept in bounds


def test_pool_gather_bitexact(L):
    from paper_1711_06505_b200.pool import ImagePool
    rng = np.random.default_rng(0)
    rows = rng.standard_normal((257, 4096)).astype(np.float32)
    pool = ImagePool.from_rows(rows)
    ids = rng.integers(0, 257, 1000)
    got = pool.gather(ids).cpu().numpy()
    assert np.array_equal(got, rows[ids])
    pb = ImagePool.from_rows(rows, dtype="bf16")
    gb = pb.gather(ids).cpu().numpy()
    exp = torch.as_tensor(rows[ids]).to(torch.bfloat16).float().numpy()
    assert np.array_equal(gb, exp)


def test_pool_materialize_matches_fp64_extractor(L):
    from paper_1711_06505_b200.pool import FixedExtractor, ImagePool
    rng = np.random.default_rng(1)
    lat = rng.standard_normal((64, 32)).astype(np.float32)
    ext = FixedExtractor(0x5EED, 32, 4096)
    pool = ImagePool.from_latents(lat, ext)
    got = pool.rows.cpu().numpy()
    ref = np.tanh(lat.astype(np.float64) @ ext.weight.T)  # images.py:71
    assert np.max(np.abs(got.astype(np.float64) - ref)) <= 1.2e-7  # fp64 then one fp32 rounding


def test_bucket_by_owner_stable_partition(L):
    dev = "cuda"
    rng = np.random.default_rng(5)
    for world in (1, 2, 4, 8):
        keys = np.unique(rng.integers(0, 10_000_000, 100_000)).astype(np.int32)
        n = len(keys)
        t = torch.as_tensor(keys, device=dev)
        cnt = torch.tensor([n], dtype=torch.int32, device=dev)
        send = torch.empty(n, dtype=torch.int32, device=dev)
        counts = torch.empty(world, dtype=torch.int32, device=dev)
        perm = torch.empty(n, dtype=torch.int32, device=dev)
        perm_inv = torch.empty(n, dtype=torch.int32, device=dev)
        ws = torch.empty(L.lib.dicm_bucket_workspace(n, world), dtype=torch.uint8, device=dev)
        L.check(L.lib.dicm_bucket_by_owner(t.data_ptr(), cnt.data_ptr(), n, world, send.data_ptr(), counts.data_ptr(),
                                           perm.data_ptr(), perm_inv.data_ptr(), ws.data_ptr(), ws.numel(),
                                           L.stream_handle()))
        torch.cuda.synchronize()
        owner = keys % world
        exp_counts = np.bincount(owner, minlength=world)
        assert np.array_equal(counts.cpu().numpy(), exp_counts)
        order = np.argsort(owner, kind="stable")
        assert np.array_equal(send.cpu().numpy(), (keys[order] // world))
        p = perm.cpu().numpy()
        assert np.array_equal(np.sort(p), np.arange(n))
        assert np.array_equal(p[order], np.arange(n))
        assert np.array_equal(perm_inv.cpu().numpy()[p], np.arange(n))  # the gather form of perm


def test_counter_based_table_init_is_rank_invariant():
    """dicm_table_init: a row's values depend on (key, row) only -- the shards
    of world 3 interleave to the world-1 table -- and follow 0.05 N(0,1)
    (reference model.py:316-319)."""
    from paper_1711_06505_b200 import _lib as L
    V, d, key = 100_003, 12, (7 << 32) | 12345
    full = torch.empty((V, d), device="cuda")
    L.check(L.lib.dicm_table_init(full.data_ptr(), V, d, 1, 0, V, key, 0.05, L.stream_handle()))
    world = 3
    for r in range(world):
        n_local = -(-V // world)
        t = torch.full((n_local, d), float("nan"), device="cuda")
        L.check(L.lib.dicm_table_init(t.data_ptr(), n_local, d, world, r, V, key, 0.05, L.stream_handle()))
        mine = full[r::world]
        assert torch.equal(t[:len(mine)], mine)
        assert torch.count_nonzero(t[len(mine):]) == 0
    x = full.double()
    assert abs(x.mean().item()) < 1e-3 and abs(x.std().item() - 0.05) < 1e-3


@pytest.mark.parametrize("n,keys", [(1, 1), (1000, 7), (823_296, 561_000), (200_000, 50)])
def test_ref_transpose_groups_every_reference_under_its_key(n, keys):
    """dicm_ref_transpose (counting sort of a dedup inverse): start[] is the
    exclusive prefix of the per-key counts, start[k] = n past the last key,
    and each group holds exactly its key's positions (any order)."""
    from paper_1711_06505_b200 import _lib as L
    rng = np.random.default_rng(n)
    inv = rng.integers(0, keys, n).astype(np.int32)
    inv[:min(keys, n)] = np.arange(min(keys, n))  # every key present
    cap = keys + 17
    d_inv = torch.as_tensor(inv, device="cuda")
    order = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    start = torch.full((cap + 1,), -1, dtype=torch.int32, device="cuda")
    ws = torch.empty(L.lib.dicm_ref_transpose_workspace(n, cap), dtype=torch.uint8, device="cuda")
    L.check(L.lib.dicm_ref_transpose(d_inv.data_ptr(), n, cap, ws.data_ptr(), ws.numel(), order.data_ptr(),
                                     start.data_ptr(), L.stream_handle()))
    o, st = order.cpu().numpy(), start.cpu().numpy()
    counts = np.bincount(inv, minlength=cap)
    assert np.array_equal(st[:cap], np.concatenate([[0], np.cumsum(counts)[:-1]]))
    assert st[cap] == n
    assert np.array_equal(np.sort(o), np.arange(n))
    assert np.array_equal(inv[o], np.repeat(np.arange(cap), counts))
