"""Multi-GPU plumbing for the blocked layers: minibatch sharding and the
weight-gradient allreduce.

The FC / conv / FFN layers are data parallel over the minibatch: every rank
owns a contiguous range of token (or image) blocks and there is NO data-path
collective.  Training (BASELINE cfg 5) has exactly one exchange step, the
sum-allreduce of dW, which ``GradSync`` issues per layer bucket on a side
stream as soon as that layer's dW is produced, so NCCL (NVLink / NVSwitch,
NVLS when available) runs under the remaining backward GEMMs, and runs that
layer's optimizer update on the same side stream right after its bucket
lands.  The paper's distributed runs did the same with oneCCL on CPUs
(PAPER.md:909).
"""

from __future__ import annotations

import os
from typing import Callable, Optional

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


class GradSync:
    """Per-layer gradient exchange + update on a side stream.

    For each layer bucket the caller reports two points of its (main-stream)
    backward: ``grad_ready(t)`` once the bucket's gradient ``t`` is written,
    and ``update_ready(fn)`` once nothing on the main stream reads the
    layer's weights any more (its backward-data GEMM is issued).  The side
    stream waits for the first point, sum-allreduces ``t`` (NCCL: the side
    stream then waits for the collective without blocking the host), waits
    for the second point and runs ``fn()`` — the layer's split-SGD — on the
    side stream.  ``finish()`` makes the main stream wait for all of it.

    With one rank there is nothing to exchange: the updates are queued on the
    main stream at ``finish()`` in bucket order (no second stream, identical
    results).  ``reduce_fn`` replaces the collective (tests emulate ranks
    with it)."""

    def __init__(self, group=None, reduce_fn: Optional[Callable[[torch.Tensor], None]] = None,
                 device=None):
        self.group = group
        self.reduce_fn = reduce_fn
        if group is not None:
            self.world_size = dist.get_world_size(group)
        else:
            self.world_size = world()[1]
        self.active = self.world_size > 1 or reduce_fn is not None
        self.device = device
        self.stream = torch.cuda.Stream(device=device) if (self.active and torch.cuda.is_available()) else None
        self.deferred: list[Callable[[], None]] = []
        self.issued = 0

    def _event(self) -> torch.cuda.Event:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        return ev

    def _reduce(self, t: torch.Tensor) -> None:
        if self.reduce_fn is not None:
            self.reduce_fn(t)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def grad_ready(self, t: torch.Tensor) -> None:
        if not self.active:
            return
        self.issued += 1
        if self.stream is None:  # host tensors (gloo on CPU): in program order
            self._reduce(t)
            return
        ev = self._event()
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(ev)
            self._reduce(t)

    def update_ready(self, fn: Callable[[], None]) -> None:
        if not self.active:
            self.deferred.append(fn)
            return
        if self.stream is None:
            fn()
            return
        ev = self._event()
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(ev)
            fn()

    def finish(self) -> None:
        if not self.active:
            for fn in self.deferred:
                fn()
            self.deferred.clear()
            return
        if self.stream is not None:
            torch.cuda.current_stream(self.device).wait_stream(self.stream)


def allreduce_sweep(sizes_bytes, dtype=torch.bfloat16, iters: int = 20, group=None):
    """Device time (ms, max over ranks) of one sum-allreduce per buffer size:
    the measurement that sizes the gradient buckets."""
    out = {}
    for nbytes in sizes_bytes:
        t = torch.ones(max(1, nbytes // torch.tensor([], dtype=dtype).element_size()), dtype=dtype,
                       device="cuda")
        for _ in range(3):
            dist.all_reduce(t, group=group)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            dist.all_reduce(t, group=group)
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / iters], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX, group=group)
        out[int(nbytes)] = float(ms.item())
    return out


def init_from_env(backend: Optional[str] = None):
    """torchrun-style init (RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT).
    NCCL on CUDA (high-priority communication streams, so the collective's
    CTAs are scheduled ahead of queued GEMM CTAs), gloo otherwise; returns
    (rank, world_size)."""
    if int(os.environ.get("WORLD_SIZE", "1")) <= 1:
        return 0, 1
    if not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        kw = {}
        if backend == "nccl":
            local = int(os.environ.get("LOCAL_RANK", "0"))
            if os.environ.get("TPP_BENCH_ONE_GPU") != "1":
                torch.cuda.set_device(local)
            kw["device_id"] = torch.device("cuda", local)
            try:
                kw["pg_options"] = dist.ProcessGroupNCCL.Options(is_high_priority_stream=True)
            except Exception:
                pass
        dist.init_process_group(backend, **kw)
    return dist.get_rank(), dist.get_world_size()
