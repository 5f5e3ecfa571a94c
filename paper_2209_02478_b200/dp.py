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

from .trainer import _DevArray


def rank_sizes(dist: str, iterations: int, base_seed: int, rank: int) -> List[int]:
    """Per-rank sequence lengths: the reference sampler with seed base + rank."""
    from .planner import host_lib
    return [int(s) for s in host_lib().workload(dist, 1, iterations, base_seed + rank)]


def rank_sizes_grouped(dist: str, iterations: int, base_seed: int, rank: int,
                       jitter: float = 0.05) -> List[int]:
    """Length-grouped per-rank sequence lengths: every step's length group is
    the reference sampler's size (seed base, shared by all ranks); each rank
    draws its own S within +-jitter of it from its own RNG and clamps to the
    distribution's [LO, HI] (the last two fields of the spec). Ranks train
    different lengths under their own plans without every step waiting for
    the longest of N independent draws (HF Trainer group_by_length)."""
    from .planner import host_lib
    shared = [int(s) for s in host_lib().workload(dist, 1, iterations, base_seed)]
    f = dist.split(":")
    lo, hi = int(f[-2]), int(f[-1])
    g = np.random.default_rng(base_seed + 7919 * (rank + 1))
    u = g.uniform(-jitter, jitter, size=len(shared))
    return [int(min(hi, max(lo, round(s * (1.0 + d))))) for s, d in zip(shared, u)]


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

    def _exchange(self, stream):
        if getattr(self.tr, "_dp", None) is not None:
            raise RuntimeError("trainer has a NativeDP attached: gradients would be reduced "
                               "(and scaled by 1/world) twice")
        if self.world > 1:
            import torch
            # the all-reduce runs on torch's current stream: order it behind
            # the backward issued on `stream`
            if stream is not None and torch.cuda.is_available():
                s = stream if isinstance(stream, torch.cuda.Stream) else \
                    torch.cuda.ExternalStream(stream)
                with torch.cuda.stream(s):
                    self._allreduce(self.grads())
            else:
                self._allreduce(self.grads())

    def step(self, tokens, types, labels, stream=None) -> dict:
        row = self.tr.step(tokens, types, labels, optimizer=False, stream=stream)
        self._exchange(stream)
        self.tr.optimizer_step(1.0 / self.world, stream=stream)
        return row

    def step_device(self, batch, stream=None) -> dict:
        row = self.tr.step_device(batch, optimizer=False, stream=stream)
        self._exchange(stream)
        self.tr.optimizer_step(1.0 / self.world, stream=stream)
        return row


class NativeDP:
    """The library's own NCCL communicator (C ABI mimose_dp_*).

    Rank 0 makes the NCCL unique id; it is broadcast over the already
    initialised torch.distributed group (any backend: it is 128 host bytes).
    Attach to a Trainer with ``trainer.attach_dp(dp, bucket_mb)``: gradients
    are then summed in buckets on the communicator's high-priority stream as
    the backward finishes each block (overlapping the remaining backward),
    and the optimizer waits for the last bucket and scales by 1/world.
    """

    def __init__(self, device: int, rank: int, world: int, group=None, unique_id: bytes = None,
                 reduce_fn: Optional[Callable] = None):
        """reduce_fn(tensor, op, stream) -> None: custom transport instead of
        NCCL (tensor = CUDA view of the bucket, op 'sum' / 'max', stream =
        torch.cuda.ExternalStream of the communicator's stream, already
        ordered behind the backward that produced the bucket); it must leave
        the cross-rank result in `tensor`."""
        import ctypes as C
        from ._lib import DP_REDUCE, check, cuda_lib
        self.lib = cuda_lib()
        self.rank, self.world = rank, world
        self.reduce_calls = 0
        if reduce_fn is not None:
            import torch

            def _cb(user, buf, n, dtype, op, stream):
                try:
                    typestr = "<f4" if dtype == 0 else "<i2"
                    t = torch.as_tensor(_DevArray(buf, n, typestr), device="cuda")
                    if dtype == 1:
                        t = t.view(torch.bfloat16)
                    reduce_fn(t, "max" if op == 1 else "sum",
                              torch.cuda.ExternalStream(stream, device=torch.device("cuda", device)))
                    self.reduce_calls += 1
                    return 0
                except Exception as e:  # noqa: BLE001 - reported through the C status
                    self.error = e
                    return 1
            self._cb = DP_REDUCE(_cb)
            h = C.c_void_p()
            check(self.lib.mimose_dp_create_custom(int(device), int(rank), int(world), self._cb,
                                                   None, C.byref(h)))
            self.handle = h
            return
        if unique_id is None:
            buf = (C.c_char * 128)()
            if rank == 0:
                check(self.lib.mimose_dp_unique_id(buf))
            unique_id = bytes(buf)
            if world > 1:
                import torch.distributed as dist
                obj = [unique_id]
                dist.broadcast_object_list(obj, src=0, group=group)
                unique_id = obj[0]
        uid = (C.c_char * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        check(self.lib.mimose_dp_create(int(device), uid, int(rank), int(world), C.byref(h)))
        self.handle = h

    def device_bytes(self) -> int:
        """Device memory the NCCL communicator holds outside the budget arena."""
        import ctypes as C
        from ._lib import check
        out = C.c_int64()
        check(self.lib.mimose_dp_device_bytes(self.handle, C.byref(out)))
        return out.value

    def allreduce_(self, tensor, op: str = "sum", stream=None):
        """In-place all-reduce of a CUDA fp32 / bf16 tensor on `stream`."""
        import torch
        from ._lib import check
        dt = {torch.float32: 0, torch.bfloat16: 1}[tensor.dtype]
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        check(self.lib.mimose_dp_allreduce(self.handle, tensor.data_ptr(), tensor.numel(), dt,
                                           {"sum": 0, "max": 1}[op], s))
        return tensor

    def close(self):
        if getattr(self, "handle", None):
            self.lib.mimose_dp_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def timed(fn, *args, **kw):
    t0 = time.perf_counter()
    out = fn(*args, **kw)
    return out, time.perf_counter() - t0
