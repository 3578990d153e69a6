"""Multi-GPU plumbing for the blocked layers: minibatch sharding and the
weight-gradient allreduce.

The FC / conv / FFN layers are data parallel over the minibatch: every rank
owns a contiguous range of token (or image) blocks and there is NO data-path
collective.  Training (BASELINE cfg 5) has exactly one exchange step, the
sum-allreduce of dW, which ``GradAllreduce`` issues per layer bucket as soon
as that layer's dW is produced, so NCCL (NVLink / NVSwitch, NVLS when
available) runs on its own stream under the remaining backward GEMMs.  The
paper's distributed runs did the same with oneCCL on CPUs.
"""

from __future__ import annotations

import os
from typing import Optional

import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    """(rank, world_size) of the default group, (0, 1) when not initialised."""
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_range(total_blocks: int, world_size: int, rank: int) -> tuple[int, int]:
    """Contiguous block range [start, start + count) of ``rank``; the first
    ``total % world`` ranks take one extra block."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad rank / world size")
    base, extra = divmod(total_blocks, world_size)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


class GradAllreduce:
    """Bucketed, overlapped sum-allreduce of gradient buffers.

    ``push(t)`` enqueues an async allreduce of ``t`` ordered after the work
    already on the current stream (NCCL's stream waits on it), and returns
    immediately so the caller keeps launching backward GEMMs; ``wait()``
    makes the current stream wait for every pending bucket (before the
    optimizer step).  With one rank it is a no-op."""

    def __init__(self, group=None, bucket_bytes: int = 0):
        self.group = group
        self.bucket_bytes = bucket_bytes
        self.pending = []
        r, w = world()
        self.world_size = w if group is None else dist.get_world_size(group)

    def push(self, t: torch.Tensor) -> None:
        if self.world_size == 1:
            return
        if self.bucket_bytes and t.numel() * t.element_size() > self.bucket_bytes:
            step = max(1, self.bucket_bytes // t.element_size())
            for i in range(0, t.numel(), step):
                self.pending.append(dist.all_reduce(t[i:i + step], op=dist.ReduceOp.SUM,
                                                    group=self.group, async_op=True))
            return
        self.pending.append(dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group,
                                            async_op=True))

    def wait(self) -> None:
        for w in self.pending:
            w.wait()
        self.pending.clear()


def init_from_env(backend: Optional[str] = None):
    """torchrun-style init (RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT).
    NCCL on CUDA, gloo otherwise; returns (rank, world_size)."""
    if int(os.environ.get("WORLD_SIZE", "1")) <= 1:
        return 0, 1
    if not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        kw = {}
        if backend == "nccl":
            local = int(os.environ.get("LOCAL_RANK", "0"))
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend, **kw)
    return dist.get_rank(), dist.get_world_size()
