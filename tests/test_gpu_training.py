"""GPU parity of the training-side BRGEMMs (backward-data with fused RELU_INV,
backward-weights via MN-major tcgen05 operands), the softmax-CE gradient and
one full blocked-MLP training step, against the CPU oracle composition of the
reference TPPs.  BF16 layers: normwise <= 2e-2 (north_star tolerance)."""

import numpy as np
import pytest
import torch

from oracle import tpp_oracle as O

from gpu_util import bf16_bits_to_f32, normwise, to_dev, to_host

pytestmark = pytest.mark.gpu
tpp = pytest.importorskip("paper_2104_05755_b200")
from paper_2104_05755_b200 import training as T  # noqa: E402

TOL = 2e-2


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield
    torch.cuda.synchronize()


def _blocked(x_logical: np.ndarray, bn: int) -> np.ndarray:
    """[T, D] -> blocked [T/bn][D/64][bn][64]."""
    t, d = x_logical.shape
    return x_logical.reshape(t // bn, bn, d // 64, 64).transpose(0, 2, 1, 3).copy()


def _logical(blocked: np.ndarray) -> np.ndarray:
    nb, db, bn, b = blocked.shape
    return blocked.transpose(0, 2, 1, 3).reshape(nb * bn, db * b)


def _bf16(rng, shape, std):
    return O.fp32_to_bf16_rne((rng.standard_normal(shape) * std).astype(np.float32))


@pytest.mark.parametrize("bn", [64, 32])
def test_fc_backward_data_relu_inv(bn):
    rng = np.random.default_rng(50)
    T_, I_, O_ = 256, 256, 384
    w = _bf16(rng, (O_, I_), 0.05)                     # logical [out, in]
    dy = _bf16(rng, (T_, O_), 1.0)
    mask = rng.random((T_, I_)) > 0.4
    layer = tpp.FcLayer(O_ // 64, I_ // 64, 64, 64, None,
                        w_packed=to_dev(T.pack_logical_weight(torch.from_numpy(w.view(np.int16))).numpy().view(np.uint16)))
    mask_bytes = np.packbits(_blocked(mask.astype(np.uint8), bn), axis=-1, bitorder="little")
    out = layer.backward_data(to_dev(_blocked(dy, bn)), T_ // bn, bn, relu_mask_in=to_dev(mask_bytes))
    got = bf16_bits_to_f32(_logical(to_host(out).reshape(T_ // bn, I_ // 64, bn, 64)))
    ref = O.blocked_matmul(O.bf16_to_fp32(dy), O.bf16_to_fp32(w).T.copy())
    ref = O.round_bf16(O.relu_inv(ref, mask))
    assert normwise(got, ref) <= TOL
    assert np.all(got[~mask] == 0)


def test_fc_backward_weights():
    rng = np.random.default_rng(51)
    T_, I_, O_ = 512, 192, 256
    x = _bf16(rng, (T_, I_), 1.0)
    dy = _bf16(rng, (T_, O_), 1.0)
    layer = tpp.FcLayer(O_ // 64, I_ // 64, 64, 64, None,
                        w_packed=torch.zeros(O_ * I_, dtype=torch.bfloat16, device="cuda"))
    dw = layer.backward_weights(to_dev(_blocked(dy, 64)), to_dev(_blocked(x, 64)), T_ // 64, 64)
    got = T.unpack_weight(dw.cpu(), O_, I_).numpy()
    ref = O.blocked_matmul(O.bf16_to_fp32(dy).T.copy(), O.bf16_to_fp32(x).T.copy())
    assert normwise(got, ref) <= 1e-5  # FP32 output; only the summation order differs


def _blocked_b(x_logical: np.ndarray, bn: int, bm: int) -> np.ndarray:
    """[T, D] -> blocked [T/bn][D/bm][bn][bm]."""
    t, d = x_logical.shape
    return x_logical.reshape(t // bn, bn, d // bm, bm).transpose(0, 2, 1, 3).copy()


# (tokens, classes, bn, bm): 128 tokens run the 16-token kernel, >= 148 tokens
# the pipelined persistent one (one or several sub-batches per SM, classes not
# a multiple of 16, tokens per SM not a multiple of the sub-batch)
@pytest.mark.parametrize("T_,C_,bn,bm", [(128, 256, 64, 64), (640, 1024, 64, 64), (2048, 1024, 64, 64),
                                          (9216, 1024, 64, 64), (2048, 1024, 32, 64), (1216, 512, 64, 64),
                                          (320, 192, 32, 32), (448, 200, 64, 40)])
def test_softmax_xent_matches_reference_softmax(T_, C_, bn, bm):
    rng = np.random.default_rng(52)
    logits = (rng.standard_normal((T_, C_)) * 3).astype(np.float32)
    logits[5, 7] = np.float32(np.nan) if T_ > 300 else logits[5, 7]   # a NaN row: NaN max, NaN outputs
    tg = rng.integers(0, C_, T_).astype(np.int32)
    d, loss = tpp.softmax_xent_blocked(to_dev(_blocked_b(logits, bn, bm)), to_dev(tg), T_ // bn, C_ // bm, bn, bm,
                                       1.0 / 1000)
    got = _logical(to_host(d).reshape(T_ // bn, C_ // bm, bn, bm))
    p = np.stack([O.softmax_slice(logits[i:i + 1])[0] for i in range(T_)])
    onehot = np.zeros_like(p)
    onehot[np.arange(T_), tg] = 1
    want = O.fp32_to_bf16_rne((p - onehot) * np.float32(1e-3))
    nan_w, nan_g = (want & 0x7FFF) > 0x7F80, (got & 0x7FFF) > 0x7F80
    assert np.array_equal(nan_g, nan_w)  # NaN payloads differ between CPU and GPU
    assert np.array_equal(got[~nan_w], want[~nan_w])  # bitwise: same softmax order, same RNE
    ref_loss = -np.log(p[np.arange(T_), tg])
    assert np.allclose(to_host(loss), ref_loss, rtol=1e-5, atol=1e-6, equal_nan=True)


def test_mlp_train_step_vs_oracle():
    rng = np.random.default_rng(53)
    dims = [128, 256, 256, 128]
    T_ = 256
    ws = [(rng.standard_normal((dims[l + 1], dims[l])) * 0.05).astype(np.float32) for l in range(3)]
    x = _bf16(rng, (T_, dims[0]), 1.0)
    tg = rng.integers(0, dims[-1], T_).astype(np.int32)
    mlp = tpp.BlockedMLP(dims, T_, bn=64, lr=0.5, global_batch=T_,
                         weights=[torch.from_numpy(w) for w in ws], fuse_sgd=False)
    loss = mlp.train_step(to_dev(_blocked(x, 64)), to_dev(tg))
    torch.cuda.synchronize()
    new_ref, dws_ref, loss_ref = O.mlp_train_step(x, ws, tg, 0.5, T_)
    assert np.allclose(to_host(loss), loss_ref, rtol=2e-2, atol=1e-3)
    for l in range(3):
        dw = T.unpack_weight(mlp.dw[l].cpu(), dims[l + 1], dims[l]).numpy()
        assert normwise(dw, dws_ref[l]) <= TOL, l
        got_w = mlp.master_weight(l).cpu().numpy()
        assert normwise(got_w - ws[l], new_ref[l] - ws[l]) <= TOL, l
    # split-SGD fused into the backward-weights epilogue: bitwise the same step
    fused = tpp.BlockedMLP(dims, T_, bn=64, lr=0.5, global_batch=T_, weights=[torch.from_numpy(w) for w in ws])
    assert fused.fuse_sgd
    fused.train_step(to_dev(_blocked(x, 64)), to_dev(tg))
    torch.cuda.synchronize()
    for l in range(3):
        assert torch.equal(fused.hi[l].view(torch.int16), mlp.hi[l].view(torch.int16)), l
        assert torch.equal(fused.lo[l], mlp.lo[l]), l


# ---------------------------------------------------------------------------
# data parallelism: a sharded step equals the global-batch step
# ---------------------------------------------------------------------------

def _mlp_case(seed=60):
    rng = np.random.default_rng(seed)
    dims = [128, 256, 256, 128]
    T_ = 512
    ws = [(rng.standard_normal((dims[l + 1], dims[l])) * 0.05).astype(np.float32) for l in range(3)]
    x = _bf16(rng, (T_, dims[0]), 1.0)
    tg = rng.integers(0, dims[-1], T_).astype(np.int32)
    return dims, T_, ws, x, tg


@pytest.mark.parametrize("grad_dtype", ["fp32", "bf16"])
def test_sharded_step_equals_global_step_emulated(grad_dtype):
    """Two emulated ranks (half the tokens each, loss scaled by the global
    batch) whose dW buckets are summed before split-SGD reproduce the
    single-rank global-batch step."""
    dims, T_, ws, x, tg = _mlp_case()
    lr = 0.5
    wt = [torch.from_numpy(w) for w in ws]
    full = tpp.BlockedMLP(dims, T_, bn=64, lr=lr, global_batch=T_, weights=wt, fuse_sgd=False)
    full.train_step(to_dev(_blocked(x, 64)), to_dev(tg))
    half = T_ // 2
    shards = [tpp.BlockedMLP(dims, half, bn=64, lr=lr, global_batch=T_, weights=wt, grad_dtype=grad_dtype,
                             fuse_sgd=False) for _ in range(2)]
    for r, m in enumerate(shards):
        m.forward(to_dev(_blocked(x[r * half:(r + 1) * half], 64)))
        m.backward(to_dev(tg[r * half:(r + 1) * half]))
    for l in range(3):                                    # the allreduce(sum)
        s = shards[0].dw[l] + shards[1].dw[l]
        for m in shards:
            m.dw[l].copy_(s)
    for m in shards:
        m.step()
    torch.cuda.synchronize()
    # forward activations are row-independent: bitwise equal to the global run
    for r, m in enumerate(shards):
        for l in range(1, 3):
            a = full.h[l].reshape(T_ // 64, -1)[r * (half // 64):(r + 1) * (half // 64)].reshape(-1)
            assert torch.equal(a.view(torch.int16), m.h[l].view(torch.int16)), (r, l)
    tol_dw = 1e-5 if grad_dtype == "fp32" else TOL
    for l in range(3):
        got = shards[0].dw[l].float().cpu().numpy()
        assert normwise(got, full.dw[l].cpu().numpy()) <= tol_dw, l
        w0 = ws[l]
        d_full = full.master_weight(l).cpu().numpy() - w0
        for m in shards:
            assert normwise(m.master_weight(l).cpu().numpy() - w0, d_full) <= tol_dw, l
        assert torch.equal(shards[0].hi[l].view(torch.int16), shards[1].hi[l].view(torch.int16))


def _dp_worker(rank, ws_, port, grad_dtype, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws_))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=ws_)
    try:
        import paper_2104_05755_b200 as tp
        dims, T_, ws, x, tg = _mlp_case()
        half = T_ // ws_
        m = tp.BlockedMLP(dims, half, bn=64, lr=0.5, global_batch=T_, weights=[torch.from_numpy(w) for w in ws],
                          grad_dtype=grad_dtype)
        assert m.sync.active and m.sync.stream is not None
        m.train_step(to_dev(_blocked(x[rank * half:(rank + 1) * half], 64)), to_dev(tg[rank * half:(rank + 1) * half]))
        torch.cuda.synchronize()
        q.put((rank, [m.master_weight(l).cpu().numpy() for l in range(3)], m.sync.issued))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("grad_dtype", ["fp32", "bf16"])
def test_sharded_step_two_processes_gloo(grad_dtype):
    """The real exchange path: 2 processes (both on cuda:0, gloo — collectives
    wait on the host, no kernel waits on another), GradSync's side stream
    all-reducing each dW bucket and running that layer's split-SGD after it.
    Both ranks end with the same weights as the global-batch step."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, grad_dtype, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(2)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    dims, T_, ws, x, tg = _mlp_case()
    full = tpp.BlockedMLP(dims, T_, bn=64, lr=0.5, global_batch=T_, weights=[torch.from_numpy(w) for w in ws])
    full.train_step(to_dev(_blocked(x, 64)), to_dev(tg))
    torch.cuda.synchronize()
    tol = 1e-5 if grad_dtype == "fp32" else TOL
    for rank, wts, issued in res:
        assert issued == 3
        for l in range(3):
            d_full = full.master_weight(l).cpu().numpy() - ws[l]
            assert normwise(wts[l] - ws[l], d_full) <= tol, (rank, l)
    for l in range(3):
        assert np.array_equal(res[0][1][l], res[1][1][l])
