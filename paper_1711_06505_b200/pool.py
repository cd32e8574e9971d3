"""The image pool: 4096-d feature rows resident in HBM.

The reference keeps float32 latents and runs the frozen extractor on every
lookup (``ImageFeatureStore.raw_features`` images.py:99-101 ->
``FixedExtractor.extract`` images.py:62-71).  On B200 the extractor output is
materialized once -- computed in fp64 on the device by
``dicm_pool_materialize`` and rounded to the pool dtype -- and the hot path
reads rows straight from HBM.  Row ids are the image ids; a sharded pool
(multi-GPU) holds the rows ``id % world == rank`` at local row ``id // world``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L


class FixedExtractor:
    """Frozen latent -> feature map tanh(z R^T) (reference images.py:48-71);
    same seeded R as the reference."""

    def __init__(self, seed, latent_dim, out_dim):
        self.seed = int(seed)
        self.latent_dim = int(latent_dim)
        self.out_dim = int(out_dim)
        rng = np.random.default_rng(self.seed)
        self.weight = rng.normal(0.0, 1.0 / np.sqrt(latent_dim), (out_dim, latent_dim))


_DT = {"fp32": (torch.float32, L.POOL_F32), "bf16": (torch.bfloat16, L.POOL_BF16)}


class ImagePool:
    """Device-resident rows [n, d_raw] in fp32 or bf16."""

    def __init__(self, rows, world=1, rank=0, global_size=None):
        if rows.dim() != 2 or not rows.is_cuda:
            raise ValueError("ImagePool expects a 2-D CUDA tensor")
        if rows.dtype not in (torch.float32, torch.bfloat16):
            raise ValueError(f"pool dtype {rows.dtype} not supported (fp32 or bf16)")
        self.rows = rows.contiguous()
        self.world, self.rank = int(world), int(rank)
        self.global_size = int(global_size if global_size is not None else rows.shape[0])

    @property
    def dtype_name(self):
        return "fp32" if self.rows.dtype == torch.float32 else "bf16"

    @property
    def dtype_code(self):
        return L.POOL_F32 if self.rows.dtype == torch.float32 else L.POOL_BF16

    @property
    def d_raw(self):
        return self.rows.shape[1]

    def __len__(self):
        return self.global_size

    @property
    def local_rows(self):
        return self.rows.shape[0]

    @classmethod
    def from_rows(cls, rows, dtype="fp32", device="cuda", world=1, rank=0):
        """``rows``: the GLOBAL [P, d_raw] matrix; a sharded pool keeps rows
        id % world == rank (reference placement: shard_of, runtime.py:60-68)."""
        tdt, _ = _DT[dtype]
        rows = np.asarray(rows, dtype=np.float32)
        t = torch.as_tensor(rows[rank::world]).to(device=device, dtype=tdt)
        return cls(t, world, rank, rows.shape[0])

    @classmethod
    def from_latents(cls, latents, extractor, dtype="fp32", device="cuda", world=1, rank=0,
                     chunk_rows=1 << 16):
        """Materialize tanh(z R^T) for the rows this rank owns.  ``latents``
        is the GLOBAL [P, k] float32 matrix (host or device)."""
        tdt, code = _DT[dtype]
        lat = torch.as_tensor(latents, dtype=torch.float32)
        P = lat.shape[0]
        if world > 1:
            lat = lat[rank::world]
        n = lat.shape[0]
        proj = torch.as_tensor(extractor.weight, dtype=torch.float64, device=device).contiguous()
        out = torch.empty((n, extractor.out_dim), dtype=tdt, device=device)
        s = L.stream_handle()
        for a in range(0, n, chunk_rows):
            b = min(n, a + chunk_rows)
            z = lat[a:b].to(device).contiguous()
            L.check(L.lib.dicm_pool_materialize(z.data_ptr(), proj.data_ptr(), b - a, extractor.out_dim,
                                                extractor.latent_dim, out[a:].data_ptr(), code, s))
        return cls(out, world, rank, P)

    @classmethod
    def synthetic(cls, n_rows, d_raw=4096, latent_dim=32, seed=0, dtype="fp32", device="cuda",
                  world=1, rank=0, extractor_seed=0x5EED):
        """Benchmark pool: latents ~ N(0,1)^k (reference data.py:137),
        features tanh(z R^T).  Large sharded pools draw each
        shard's latents on its own device (seeded by (seed, rank)), so a
        20M-row pool never passes through host memory."""
        ext = FixedExtractor(extractor_seed, latent_dim, d_raw)
        if world > 1 and n_rows > (1 << 22):
            n_local = len(range(rank, n_rows, world))
            gen = torch.Generator(device=device).manual_seed(seed * 1000003 + rank)
            lat = torch.randn((n_local, latent_dim), generator=gen, dtype=torch.float32, device=device)
            pool = cls.from_latents(lat, ext, dtype, device, 1, 0)
            pool.world, pool.rank, pool.global_size = world, rank, n_rows
            return pool
        gen = torch.Generator(device="cpu").manual_seed(seed)
        lat = torch.randn((n_rows, latent_dim), generator=gen, dtype=torch.float32)
        return cls.from_latents(lat, ext, dtype, device, world, rank)

    def padded(self, d_raw):
        """A copy with zero columns up to ``d_raw`` (the kernels' row width)."""
        rows = torch.zeros((self.rows.shape[0], d_raw), dtype=self.rows.dtype, device=self.rows.device)
        rows[:, :self.d_raw] = self.rows
        return ImagePool(rows, self.world, self.rank, self.global_size)

    def gather(self, ids):
        """Rows for local ids as fp32 on the device (dicm_pool_gather)."""
        ids = torch.as_tensor(np.asarray(ids, dtype=np.int32), device=self.rows.device)
        n = ids.numel()
        out = torch.empty((n, self.d_raw), dtype=torch.float32, device=self.rows.device)
        cnt = torch.tensor([n], dtype=torch.int32, device=self.rows.device)
        L.check(L.lib.dicm_pool_gather(self.rows.data_ptr(), self.dtype_code, self.d_raw, ids.data_ptr(),
                                       cnt.data_ptr(), n, out.data_ptr(), L.stream_handle()))
        return out

    def raw_features(self, ids, extractor=None):
        """Reference-shaped accessor (images.py:99-101): fp64 host rows."""
        ids = np.asarray(ids, dtype=np.int64)
        if ids.size and (ids.min() < 0 or ids.max() >= self.local_rows):
            bad = ids[(ids < 0) | (ids >= self.local_rows)][0]
            raise KeyError(f"unknown image id {bad} (store holds 0..{self.local_rows - 1})")
        return self.gather(ids).double().cpu().numpy()
