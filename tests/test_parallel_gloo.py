"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel plumbing:
minibatch shard ranges and the bucketed dW allreduce used by BlockedMLP."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_05755_b200 import parallel


def test_shard_range_covers_exactly():
    for total in (1, 7, 16, 128):
        for ws in (1, 2, 3, 8):
            seen = []
            for r in range(ws):
                s, c = parallel.shard_range(total, ws, r)
                seen.extend(range(s, s + c))
            assert seen == list(range(total))
    with pytest.raises(ValueError):
        parallel.shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        r, w = parallel.world()
        # per-layer gradient buckets with rank-dependent contents
        grads = [torch.full((n,), float(rank + 1)) * (l + 1) for l, n in enumerate((5, 1000, 33))]
        ar = parallel.GradAllreduce(bucket_bytes=256)
        for g in grads:
            ar.push(g)
        ar.wait()
        expect = [torch.full_like(g, float(sum(range(1, ws + 1)))) * (l + 1) for l, g in enumerate(grads)]
        ok = all(torch.equal(g, e) for g, e in zip(grads, expect))
        s, c = parallel.shard_range(128, w, r)
        q.put((rank, ok, r, w, s, c))
    finally:
        dist.destroy_process_group()


def test_grad_allreduce_world2_gloo():
    ws = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, *_ in res)
    assert [(r, w) for _, _, r, w, _, _ in res] == [(0, 2), (1, 2)]
    assert [(s, c) for *_, s, c in res] == [(0, 64), (64, 64)]


def _sync_worker(rank, ws, port, q):
    """GradSync on host tensors (gloo): every bucket is summed over the ranks
    before its update callback runs, callbacks run in bucket order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        sync = parallel.GradSync()
        seen = []
        grads = [torch.full((n,), float(rank + 1) * (l + 1)) for l, n in enumerate((7, 300, 64))]
        for l in range(len(grads) - 1, -1, -1):      # backward order: last layer first
            sync.grad_ready(grads[l])
            sync.update_ready(lambda l=l: seen.append((l, float(grads[l][0]))))
        sync.finish()
        total = float(sum(range(1, ws + 1)))
        ok = seen == [(l, total * (l + 1)) for l in range(len(grads) - 1, -1, -1)]
        q.put((rank, ok, sync.issued, sync.active))
    finally:
        dist.destroy_process_group()


def test_grad_sync_world2_gloo():
    ws = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sync_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == [(0, True, 3, True), (1, True, 3, True)]


def test_grad_sync_single_rank_defers_updates_in_order():
    sync = parallel.GradSync()
    assert not sync.active
    seen = []
    t = torch.ones(3)
    for l in (2, 1, 0):
        sync.grad_ready(t)
        sync.update_ready(lambda l=l: seen.append(l))
    assert seen == []            # nothing to exchange: updates wait for finish()
    sync.finish()
    assert seen == [2, 1, 0]
    # a reduce_fn stands in for the collective (rank emulation)
    red = []
    sync = parallel.GradSync(reduce_fn=lambda x: red.append(x.clone()))
    sync.grad_ready(torch.arange(3.0))
    sync.update_ready(lambda: red.append("upd"))
    sync.finish()
    assert torch.equal(red[0], torch.arange(3.0)) and red[1] == "upd"
