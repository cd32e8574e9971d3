"""Single-GPU training: the drop-in for the reference ``LocalTrainer``
(training.py:45-106).

``train_batch`` accepts the reference's ``list[Sample]`` (encoded on the host
exactly like ``encode_batch``) or a pre-encoded ``Batch``; the step itself is
``StepEngine.step`` -- device kernels only.  Like the reference it returns the
float loss, raising ``FloatingPointError`` / ``KeyError`` for a non-finite loss
or an out-of-vocabulary id, with no parameter touched by the failed step.
``train_batch_async`` skips the host round trip and returns the device loss.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .batch import Batch, encode_batch
from .engine import StepEngine


@dataclass
class TrainConfig:
    epochs: int = 1
    batch_size: int = 256
    seed: int = 0
    lr0: float = 0.001
    lr_decay: float = 0.9
    lr_interval: int = 24000
    max_iterations: int = 0


@dataclass
class TrainLog:
    losses: list = field(default_factory=list)
    lrs: list = field(default_factory=list)


def minibatches(samples, batch_size, seed, epoch=0):
    """Deterministically shuffled batches (reference data.py:284-290)."""
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    order = np.random.default_rng([int(seed) & 0xFFFFFFFF, epoch]).permutation(len(samples))
    for start in range(0, len(samples), batch_size):
        yield [samples[i] for i in order[start:start + batch_size]]


@dataclass
class AdamStateView:
    m: np.ndarray
    v: np.ndarray
    t: object


class LocalTrainer:
    def __init__(self, model, store, cfg=None, precision="fp32"):
        self.model = model
        self.store = store
        self.cfg = cfg or TrainConfig()
        self.engine = StepEngine(model, store, precision, self.cfg.lr0, self.cfg.lr_decay, self.cfg.lr_interval)
        self.dense_names = model.worker_param_names() + model.image_param_names()

    @property
    def iteration(self):
        return self.engine.iteration

    def lr(self):
        return self.engine.lr()

    def _batch(self, samples):
        return samples if isinstance(samples, Batch) else encode_batch(samples, self.model)

    def train_batch_async(self, samples):
        return self.engine.step(self._batch(samples))

    def train_batch(self, samples):
        loss = self.engine.step(self._batch(samples))
        value = float(loss.item())
        try:
            self.engine.raise_status()
        except Exception:
            self.engine.iteration -= 1  # the reference raises before counting the step
            raise
        return value

    def run(self, train_samples, log=None):
        log = log or TrainLog()
        stop = self.cfg.max_iterations or None
        for epoch in range(self.cfg.epochs):
            for batch in minibatches(train_samples, self.cfg.batch_size, self.cfg.seed, epoch):
                log.lrs.append(self.lr())
                log.losses.append(self.train_batch(batch))
                if stop and self.iteration >= stop:
                    return log
        return log

    def run_file(self, path, log=None, prefetch=2, nthreads=0):
        """Train on a JSONL sample file (reference data.py:293-311 format) with
        the native reader and the prefetching input pipeline: same batches, in
        the same order, as ``run(read_samples(path))``."""
        from .batch import iter_minibatches, read_jsonl
        from .engine import Prefetcher
        data = read_jsonl(path, self.model.schema, nthreads)
        log = log or TrainLog()
        stop = self.cfg.max_iterations or None
        e = self.engine
        for epoch in range(self.cfg.epochs):
            for b, db in Prefetcher(e, iter_minibatches(data, self.cfg.batch_size, self.cfg.seed, epoch), prefetch):
                log.lrs.append(self.lr())
                loss = e.step_device(db)
                value = float(loss.item())
                try:
                    e.raise_status()
                except Exception:
                    e.iteration -= 1
                    raise
                log.losses.append(value)
                if stop and self.iteration >= stop:
                    return log
        return log

    def snapshot(self):
        return self.model.snapshot()

    @property
    def use_graphs(self):
        """Replay whole steps from captured CUDA graphs (one capture per batch
        layout; see StepEngine.step_graphed)."""
        return self.engine.use_graphs

    @use_graphs.setter
    def use_graphs(self, on):
        self.engine.use_graphs = bool(on)

    @property
    def dense_state(self):
        """name -> (m, v, t) host copies (checkpoint interop, reference
        training.py:54-56)."""
        e, m = self.engine, self.model
        t = e.t.cpu().numpy()
        out = {}
        for n in m.dense_names:
            out[n] = AdamStateView(m.real_view(e.m, n).double().cpu().numpy(),
                                   m.real_view(e.v, n).double().cpu().numpy(), int(t[e.span_index[n]]))
        return out

    def set_adam_state(self, name, m=None, v=None, t=None):
        """Write Adam state of one parameter into the device buffers
        (checkpoint restore, reference checkpoint.py:228-243)."""
        set_adam_state(self.engine, self.model, name, m, v, t)

    def reset_adam_state(self, name):
        """Fresh optimizer state for a re-initialised parameter."""
        reset_adam_state(self.engine, self.model, name)

    @property
    def table_state(self):
        e = self.engine
        m = self.model
        return {f: AdamStateView(m.real_table(e.tm[f]).double().cpu().numpy(),
                                 m.real_table(e.tv[f]).double().cpu().numpy(),
                                 e.tt[f].cpu().numpy().astype(np.int64)) for f in e.tm}


def set_adam_state(engine, model, name, m=None, v=None, t=None):
    """Adam state of one parameter -> the engine's device buffers: dense
    parameters into the fused m / v buffers and the per-span step counter,
    tables into the per-row m / v / t (a sharded engine takes its local rows)."""
    import torch
    if name.startswith("id_emb/"):
        f = name.split("/", 1)[1]
        if m is not None:
            model.real_table(engine.tm[f]).copy_(torch.as_tensor(np.asarray(m), dtype=torch.float32))
        if v is not None:
            model.real_table(engine.tv[f]).copy_(torch.as_tensor(np.asarray(v), dtype=torch.float32))
        if t is not None:
            engine.tt[f].copy_(torch.as_tensor(np.asarray(t), dtype=torch.int32))
        return
    if m is not None:
        model.write_real_view(engine.m, name, m)
    if v is not None:
        model.write_real_view(engine.v, name, v)
    if t is not None:
        engine.t[engine.span_index[name]] = int(np.asarray(t))


def reset_adam_state(engine, model, name):
    if name.startswith("id_emb/"):
        f = name.split("/", 1)[1]
        engine.tm[f].zero_()
        engine.tv[f].zero_()
        engine.tt[f].zero_()
    else:
        model.dense_view(engine.m, name).zero_()
        model.dense_view(engine.v, name).zero_()
        engine.t[engine.span_index[name]] = 0
