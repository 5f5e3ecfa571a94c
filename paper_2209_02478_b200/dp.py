"""Data parallelism for the Mimose trainer.

One process per GPU. Every rank draws its own variable sequence-length
stream (reference workload.hpp sample_workload with seed = base + rank), runs
its own sheltered collection / fit / plan cache under its own budget, and
after backward the flat fp32 gradient buffer (one contiguous tensor owned by
the rank's budget arena) is summed across ranks with one all-reduce (NCCL
over NVLink on GPUs, gloo in the CPU tests); AdamW then applies
grad_scale = 1/world. Plans never cross ranks - only gradients do.

The all-reduce is the only collective on the data path; step timing is the
max over ranks (stragglers with longer sequences gate the step).
"""
from __future__ import annotations

import time
from typing import Callable, List, Optional, Sequence

import numpy as np


def rank_sizes(dist: str, iterations: int, base_seed: int, rank: int) -> List[int]:
    """Per-rank sequence lengths: the reference sampler with seed base + rank."""
    from .planner import host_lib
    return [int(s) for s in host_lib().workload(dist, 1, iterations, base_seed + rank)]


def allreduce_sum_(tensor, group=None):
    """In-place sum across ranks (NCCL for CUDA tensors, gloo for CPU)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
    return tensor


def max_over_ranks(value: float, device="cpu", group=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class DataParallelTrainer:
    """Wraps one rank's Trainer: forward/backward under the rank's own plan,
    gradient all-reduce, AdamW with 1/world scaling."""

    def __init__(self, trainer, world: int, rank: int, group=None,
                 allreduce: Optional[Callable] = None):
        self.tr = trainer
        self.world = world
        self.rank = rank
        self.group = group
        self._allreduce = allreduce or (lambda t: allreduce_sum_(t, group))
        self._grads = None

    def grads(self):
        if self._grads is None:
            self._grads = self.tr.grads()
        return self._grads

    def step(self, tokens, types, labels, stream=None) -> dict:
        row = self.tr.step(tokens, types, labels, optimizer=False, stream=stream)
        if self.world > 1:
            self._allreduce(self.grads())
        self.tr.optimizer_step(1.0 / self.world, stream=stream)
        return row

    def step_device(self, batch, stream=None) -> dict:
        row = self.tr.step_device(batch, optimizer=False, stream=stream)
        if self.world > 1:
            self._allreduce(self.grads())
        self.tr.optimizer_step(1.0 / self.world, stream=stream)
        return row


def timed(fn, *args, **kw):
    t0 = time.perf_counter()
    out = fn(*args, **kw)
    return out, time.perf_counter() - t0
