"""GPU parity: the sm_100a kernels (through the C ABI) against the reference
(golden fixtures) and the CPU oracle.  Bit-exact where the reference's order
is reproduced (ordered BRGEMM, eltwise, transforms, LayerNorm, softmax, SGD);
normwise <= 2e-2 for BF16 tensor-core layers (north_star tolerance: fp32
accumulation in a different order, then BF16 RNE)."""

import numpy as np
import pytest
import torch

from oracle import tpp_oracle as O

from gpu_util import bf16_bits_to_f32, normwise, to_dev, to_host, vnni_weights

pytestmark = pytest.mark.gpu

tpp = pytest.importorskip("paper_2104_05755_b200")

BF16_TOL = 2e-2


def bits(a):
    """Byte image of an array with every float NaN canonicalised: NaN
    payloads produced by invalid operations differ between x86 (0xFFC00000)
    and the GPU (0x7FFFFFFF); both-NaN counts as a match."""
    a = np.ascontiguousarray(np.array(a, copy=True))
    if a.dtype in (np.float32, np.float64):
        a[np.isnan(a)] = np.nan
    return a.view(np.uint8).tobytes()


def bf16_equal(a, b) -> bool:
    """BF16 pattern equality with both-NaN counted as a match."""
    a, b = np.asarray(a, np.uint16), np.asarray(b, np.uint16)
    nan = lambda p: ((p & 0x7F80) == 0x7F80) & ((p & 0x7F) != 0)  # noqa: E731
    return a.shape == b.shape and bool(np.all((a == b) | (nan(a) & nan(b))))


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield
    torch.cuda.synchronize()


# ---------------------------------------------------------------------------
# BRGEMM (ordered SIMT engine): bitwise vs the reference
# ---------------------------------------------------------------------------

def test_cfg1_brgemm_bitwise(golden):
    g = golden("cfg1_brgemm.npz")
    m = n = k = 64
    a, b = to_dev(g["a"]), to_dev(g["b"])
    c = tpp.TensorView(tpp.TensorDesc(m, n, m, tpp.DType.FP32), to_dev(g["c0"]))
    tpp.brgemm(tpp.GemmSpec(m, n, k, m, k, m, beta=1.0),
               tpp.BrgemmBatch.stride(a, b, m * k, k * n, 16), c)
    assert bits(to_host(c.primary)) == bits(g["c"])


_DT = {"fp32": "FP32", "bf16": "BF16", "fp64": "FP64", "int8": "INT8"}


@pytest.mark.parametrize("variant", ["stride", "offset", "address"])
def test_brgemm_cases_bitwise(golden, variant):
    g = golden("brgemm_cases.npz")
    for i in range(int(g["count"])):
        key = f"case{i:03d}"
        m, n, k, lda, ldb, ldc, cnt, sa, sb, vnni = (int(v) for v in g[key + "_meta"])
        dt = tpp.DType[_DT[str(g[key + "_dtype"])]]
        acc = {tpp.DType.FP64: tpp.DType.FP64, tpp.DType.INT8: tpp.DType.INT32}.get(dt, tpp.DType.FP32)
        abuf, bbuf = to_dev(g[key + "_a"]), to_dev(g[key + "_b"])
        c = tpp.TensorView(tpp.TensorDesc(m, n, ldc, acc), to_dev(g[key + "_c0"]))
        spec = tpp.GemmSpec(m, n, k, lda, ldb, ldc, in_dtype=dt, out_dtype=acc,
                            beta=float(g[key + "_beta"]),
                            a_layout=tpp.ALayout.VNNI if vnni else tpp.ALayout.PLAIN,
                            engine=tpp.Engine.ORDERED)   # the reference's order: bitwise
        if variant == "stride":
            batch = tpp.BrgemmBatch.stride(abuf, bbuf, sa, sb, cnt)
        elif variant == "offset":
            batch = tpp.BrgemmBatch.offset(abuf, bbuf, [j * sa for j in range(cnt)],
                                           [j * sb for j in range(cnt)])
        else:
            batch = tpp.BrgemmBatch.address([(abuf, j * sa) for j in range(cnt)],
                                            [(bbuf, j * sb) for j in range(cnt)])
        tpp.brgemm(spec, batch, c)
        assert bits(to_host(c.primary)) == bits(g[key + "_c"]), f"case {i} ({dt}, {variant})"


@pytest.mark.parametrize("m,n,k,count,beta", [(32, 16, 128, 37, 0.5), (32, 16, 132, 9, 1.0), (48, 24, 64, 16, 0.0)])
def test_brgemm_fp32_stride_staging_paths(m, n, k, count, beta):
    """FP32 STRIDE batches through the staged ordered engine: TMA-box staging
    (k <= 128, chunks of entries with a ragged last chunk zero-filled past
    `count`, padded lda / ldb / ldc, entry strides beyond the block) and the
    cp.async fallback (k > 128); bitwise vs the reference order."""
    rng = np.random.default_rng(100 + k + count)
    lda, ldb, ldc = m + 8, k + 4, m + 4
    sa, sb = lda * k + 8, ldb * n + 4
    af = rng.standard_normal(sa * count).astype(np.float32)
    bf = rng.standard_normal(sb * count).astype(np.float32)
    c0 = rng.standard_normal((ldc, n)).astype(np.float32)
    a_blocks = [af[i * sa: i * sa + lda * k].reshape(k, lda).T[:m, :] for i in range(count)]
    b_blocks = [bf[i * sb: i * sb + ldb * n].reshape(n, ldb).T[:k, :] for i in range(count)]
    want = O.brgemm(a_blocks, b_blocks, c0[:m, :], beta)
    c = tpp.TensorView(tpp.TensorDesc(m, n, ldc, tpp.DType.FP32),
                       torch.from_numpy(c0.T.reshape(-1).copy()).cuda())
    sp = tpp.GemmSpec(m, n, k, lda, ldb, ldc, beta=beta)
    tpp.brgemm(sp, tpp.BrgemmBatch.stride(torch.from_numpy(af).cuda(), torch.from_numpy(bf).cuda(), sa, sb, count), c)
    got = tpp.to_array(c)
    assert bits(got) == bits(np.asarray(want, dtype=np.float32)), (m, n, k, count)


@pytest.mark.parametrize("m,n,k,count,beta,variant", [
    (15, 4096, 15, 51, 0.0, "stride"), (16, 2500, 16, 33, 1.0, "stride"),
    (3, 2048, 7, 5, 0.5, "offset"), (9, 3000, 1, 64, 1.0, "address")])
def test_brgemm_fp32_narrow_column_kernel(m, n, k, count, beta, variant):
    """Narrow-and-long FP32 BRGEMMs (m, k <= 16, n >= 2048: the dilated conv's
    shape) take the one-thread-per-column ordered kernel: entries staged in
    chunks of 32 (ragged last chunk), padded lda / ldb / ldc, every batch
    addressing mode; bitwise vs the reference order."""
    rng = np.random.default_rng(7 * m + k + count)
    lda, ldb, ldc = m + 1, k + 2, m + 3
    sa, sb = lda * k + 5, ldb * n + 3
    af = rng.standard_normal(sa * count).astype(np.float32)
    bf = rng.standard_normal(sb * count).astype(np.float32)
    c0 = rng.standard_normal((ldc, n)).astype(np.float32)
    a_blocks = [af[i * sa: i * sa + lda * k].reshape(k, lda).T[:m, :] for i in range(count)]
    b_blocks = [bf[i * sb: i * sb + ldb * n].reshape(n, ldb).T[:k, :] for i in range(count)]
    want = O.brgemm(a_blocks, b_blocks, c0[:m, :], beta)
    c = tpp.TensorView(tpp.TensorDesc(m, n, ldc, tpp.DType.FP32),
                       torch.from_numpy(c0.T.reshape(-1).copy()).cuda())
    sp = tpp.GemmSpec(m, n, k, lda, ldb, ldc, beta=beta)
    ad, bd = torch.from_numpy(af).cuda(), torch.from_numpy(bf).cuda()
    if variant == "stride":
        batch = tpp.BrgemmBatch.stride(ad, bd, sa, sb, count)
    elif variant == "offset":
        batch = tpp.BrgemmBatch.offset(ad, bd, [i * sa for i in range(count)], [i * sb for i in range(count)])
    else:
        batch = tpp.BrgemmBatch.address([(ad, i * sa) for i in range(count)], [(bd, i * sb) for i in range(count)])
    tpp.brgemm(sp, batch, c)
    got = tpp.to_array(c)
    assert bits(got) == bits(np.asarray(want, dtype=np.float32)), (m, n, k, count, variant)


@pytest.mark.parametrize("m,n,k,count,sh,beta", [
    (15, 5000, 15, 51, 8, 0.0), (5, 2048, 3, 9, 0, 0.5), (16, 2049, 7, 20, 3, 1.0), (9, 70001, 15, 4, 1, 1.0)])
def test_brgemm_fp32_sliding_window_kernel(m, n, k, count, sh, beta):
    """STRIDE batches whose B blocks are overlapping column windows of one
    matrix (ldb == k odd, stride_b = sh columns: the dilated conv's taps) take
    the window kernel that stages the union once per CTA: evenly split
    columns (ragged last CTA), one or two row groups, sh = 0 (every entry the
    same window); bitwise vs the reference order."""
    rng = np.random.default_rng(11 * m + k + sh)
    lda, ldc = m + 2, m + 1
    sa = lda * k + 3
    af = rng.standard_normal(sa * count).astype(np.float32)
    wcols = n + (count - 1) * sh
    bf = rng.standard_normal(k * wcols).astype(np.float32)
    c0 = rng.standard_normal((ldc, n)).astype(np.float32)
    bm = bf.reshape(wcols, k).T
    a_blocks = [af[i * sa: i * sa + lda * k].reshape(k, lda).T[:m, :] for i in range(count)]
    b_blocks = [bm[:, i * sh: i * sh + n] for i in range(count)]
    want = O.brgemm(a_blocks, b_blocks, c0[:m, :], beta)
    c = tpp.TensorView(tpp.TensorDesc(m, n, ldc, tpp.DType.FP32),
                       torch.from_numpy(c0.T.reshape(-1).copy()).cuda())
    sp = tpp.GemmSpec(m, n, k, lda, k, ldc, beta=beta)
    tpp.brgemm(sp, tpp.BrgemmBatch.stride(torch.from_numpy(af).cuda(), torch.from_numpy(bf).cuda(),
                                          sa, sh * k, count), c)
    got = tpp.to_array(c)
    assert bits(got) == bits(np.asarray(want, dtype=np.float32)), (m, n, k, count, sh)


def test_brgemm_cancellation_and_doubling():
    """test_gemm.py:117-137 properties on the GPU (FP64, exact)."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal((6, 6))
    b = rng.standard_normal((6, 6))
    av, nav, bv = (tpp.from_array(x) for x in (a, -a, b))
    c = tpp.alloc(tpp.TensorDesc(6, 6, 6, tpp.DType.FP64))
    sp = tpp.GemmSpec(6, 6, 6, 6, 6, 6, in_dtype=tpp.DType.FP64, out_dtype=tpp.DType.FP64)
    tpp.brgemm(sp, tpp.BrgemmBatch.address([av, nav], [bv, bv]), c)
    assert np.all(tpp.to_array(c) == 0.0)
    c2 = tpp.alloc(tpp.TensorDesc(6, 6, 6, tpp.DType.FP64))
    tpp.brgemm(sp, tpp.BrgemmBatch.address([av, av], [bv, bv]), c2)
    c1 = tpp.alloc(tpp.TensorDesc(6, 6, 6, tpp.DType.FP64))
    tpp.gemm(sp, av, bv, c1)
    assert bits(tpp.to_array(c2)) == bits(2.0 * tpp.to_array(c1))


def test_brgemm_empty_batch_and_errors():
    sp = tpp.GemmSpec(2, 2, 2, 2, 2, 2, beta=1.0)
    c = tpp.from_array(np.full((2, 2), 7.0, np.float32))
    tpp.brgemm(sp, tpp.BrgemmBatch.address([], []), c)
    assert np.all(tpp.to_array(c) == 7.0)
    tpp.brgemm(tpp.GemmSpec(2, 2, 2, 2, 2, 2, beta=0.0), tpp.BrgemmBatch.address([], []), c)
    assert np.all(tpp.to_array(c) == 0.0)
    a = tpp.from_array(np.ones((2, 2), np.float32))
    with pytest.raises(tpp.TensorError):
        tpp.gemm(tpp.GemmSpec(2, 2, 2, 2, 2, 2), a, a, a)  # C aliases an input
    with pytest.raises(tpp.TensorError):
        tpp.gemm(tpp.GemmSpec(2, 2, 4, 2, 4, 2), a, a, tpp.alloc(tpp.TensorDesc(2, 2, 2, tpp.DType.FP32)))


def test_brgemm_int8_no_saturation():
    a = tpp.from_array(np.full((1, 300), 127, np.int8))
    b = tpp.from_array(np.full((300, 1), 127, np.int8))
    c = tpp.alloc(tpp.TensorDesc(1, 1, 1, tpp.DType.INT32))
    tpp.gemm(tpp.GemmSpec(1, 1, 300, 1, 300, 1, in_dtype=tpp.DType.INT8, out_dtype=tpp.DType.INT32), a, b, c)
    assert int(c.item()) == 127 * 127 * 300


# ---------------------------------------------------------------------------
# elementwise / transform / conversion TPPs: bitwise
# ---------------------------------------------------------------------------

def test_rne_convert_bitwise(golden):
    g = golden("dtypes.npz")
    pats = g["fp32_bits"].view(np.float32)
    src = tpp.TensorView(tpp.TensorDesc(pats.size, 1, pats.size, tpp.DType.FP32), to_dev(pats))
    out = tpp.convert(src, tpp.DType.BF16)
    assert np.array_equal(to_host(out.primary), g["bf16_bits"])
    back = tpp.convert(out, tpp.DType.FP32)
    assert np.array_equal(to_host(back.primary).view(np.uint32) >> 16, g["bf16_bits"].astype(np.uint32))


def test_gelu_and_exp_bitwise(golden):
    g = golden("approx.npz")
    x = g["x"]
    xv = tpp.TensorView(tpp.TensorDesc(x.size, 1, x.size, tpp.DType.FP32), to_dev(x))
    out = tpp.alloc(xv.desc)
    tpp.apply_unary(tpp.UnaryKind.GELU, xv, out)
    assert bits(to_host(out.primary)) == bits(g["gelu"])
    xe = g["xe"]
    ev = tpp.TensorView(tpp.TensorDesc(xe.size, 1, xe.size, tpp.DType.FP32), to_dev(xe))
    eo = tpp.alloc(ev.desc)
    tpp.apply_unary(tpp.UnaryKind.EXP, ev, eo)
    assert bits(to_host(eo.primary)) == bits(g["exp"])


def test_eltwise_bitwise(golden):
    g = golden("eltwise.npz")
    x = g["x"]
    m, n = x.shape
    xv = tpp.from_array(x)
    out = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.FP32))
    tpp.apply_unary(tpp.UnaryKind.RELU, xv, out, bitmask_output=True)
    assert bits(to_host(out.primary)) == bits(g["relu"])
    assert np.array_equal(to_host(out.secondary), g["mask"])
    dyv = tpp.from_array(g["dy"])
    dyv.secondary = to_dev(g["mask"])
    dx = tpp.alloc(out.desc)
    tpp.apply_unary(tpp.UnaryKind.RELU_INV, dyv, dx)
    assert bits(to_host(dx.primary)) == bits(g["relu_inv"])
    xb = tpp.from_array(x, tpp.DType.BF16)
    gb = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.BF16))
    tpp.apply_unary(tpp.UnaryKind.GELU, xb, gb)
    assert bf16_equal(to_host(gb.primary), g["gelu_bf16"])
    dyg = tpp.from_array(g["dy"])
    dyg.secondary = xv.primary
    gi = tpp.alloc(out.desc)
    tpp.apply_unary(tpp.UnaryKind.GELU_INV, dyg, gi)
    assert bits(to_host(gi.primary)) == bits(g["gelu_inv"])
    bb = tpp.broadcast(tpp.from_array(g["bias"]), tpp.Bcast.COL, m, n)
    ad = tpp.alloc(out.desc)
    tpp.apply_binary(tpp.BinaryKind.ADD, xv, bb, ad)
    assert bits(to_host(ad.primary)) == bits(g["add_bias"])
    yv, zv = tpp.from_array(g["y"]), tpp.from_array(g["z"])
    ma = tpp.alloc(out.desc)
    tpp.apply_ternary(tpp.TernaryKind.MULADD, xv, yv, zv, ma)
    assert bits(to_host(ma.primary)) == bits(g["muladd"])
    tpp.apply_ternary(tpp.TernaryKind.NMULADD, xv, yv, zv, ma)
    assert bits(to_host(ma.primary)) == bits(g["nmuladd"])
    r1 = tpp.alloc(tpp.TensorDesc(m, 1, m, tpp.DType.FP32))
    tpp.reduce(yv, tpp.ReduceSpec(tpp.ReduceAxis.ROWS, tpp.ReduceOp.SUM), r1)
    assert bits(to_host(r1.primary)) == bits(g["rsum"])
    tpp.reduce(yv, tpp.ReduceSpec(tpp.ReduceAxis.ROWS, tpp.ReduceOp.SUM, True), r1)
    assert bits(to_host(r1.primary)) == bits(g["rsumsq"])
    cv = tpp.convert(xv, tpp.DType.BF16)
    assert np.array_equal(to_host(cv.primary), g["convert_bf16"])


def test_transforms_bitwise(golden):
    g = golden("eltwise.npz")
    for pats, want_key in ((g["pats"], "vnni"), (g["pats_odd"], "vnni_odd")):
        pv = tpp.from_array(pats, tpp.DType.BF16)
        m, k = pats.shape
        out = tpp.alloc(tpp.TensorDesc(m * 2, -(-k // 2), m * 2, tpp.DType.BF16))
        tpp.transform(pv, tpp.TransformSpec(tpp.TransformKind.VNNI, alpha=2), out)
        assert np.array_equal(tpp.bits_of(out), g[want_key])
    vn = tpp.from_array(g["vnni"], tpp.DType.BF16)
    out = tpp.alloc(tpp.TensorDesc(10 * 2, 6, 20, tpp.DType.BF16))
    tpp.transform(vn, tpp.TransformSpec(tpp.TransformKind.VNNI_TO_VNNIT, alpha=2, alpha_out=2,
                                        rows=12, cols=10), out)
    assert np.array_equal(tpp.bits_of(out), g["vnnit"])
    x = np.arange(12, dtype=np.float32).reshape(3, 4)
    t = tpp.alloc(tpp.TensorDesc(4, 3, 4, tpp.DType.FP32))
    tpp.transform(tpp.from_array(x), tpp.TransformSpec(tpp.TransformKind.TRANSPOSE), t)
    assert np.array_equal(tpp.to_array(t), x.T)


# ---------------------------------------------------------------------------
# composite kernels: bitwise
# ---------------------------------------------------------------------------

def test_layernorm_view_bitwise(golden):
    g = golden("layernorm.npz")
    for i in range(4):
        x = g[f"x{i}"]
        dt = tpp.DType[_DT[str(g[f"dtype{i}"])]]
        m, n = x.shape
        xv = tpp.from_array(x, dt) if dt is tpp.DType.FP32 else tpp.from_array(x, tpp.DType.BF16)
        gg = tpp.broadcast(tpp.from_array(g[f"g{i}"]), tpp.Bcast.ROW, m, n)
        bb = tpp.broadcast(tpp.from_array(g[f"b{i}"]), tpp.Bcast.ROW, m, n)
        out = tpp.alloc(tpp.TensorDesc(m, n, m, dt))
        mo = tpp.alloc(tpp.TensorDesc(m, 1, m, tpp.DType.FP32))
        vo = tpp.alloc(tpp.TensorDesc(m, 1, m, tpp.DType.FP32))
        tpp.layernorm(xv, gg, bb, 1e-5, out, mo, vo)
        assert bits(tpp.bits_of(out)) == bits(g[f"out{i}"]), i
        assert bits(to_host(mo.primary)) == bits(g[f"mean{i}"])
        assert bits(to_host(vo.primary)) == bits(g[f"var{i}"])


def test_softmax_and_split_sgd_bitwise(golden):
    g = golden("softmax_sgd.npz")
    for xk, yk, spec in (("x", "y", tpp.SoftmaxSpec(1, 6, 40)), ("x2", "y2", tpp.SoftmaxSpec(5, 3, 33))):
        xv = tpp.from_array(g[xk])
        yv = tpp.alloc(xv.desc)
        tpp.softmax(spec, xv, yv)
        assert bits(to_host(yv.primary)) == bits(g[yk])
    split = tpp.split_fp32(tpp.from_array(g["w0"]))
    for gi in g["grads"]:
        tpp.split_sgd_step(split, tpp.from_array(gi), float(g["lr"]))
    assert bits(tpp.to_array(tpp.pack_fp32(split))) == bits(g["w1"])


def test_fc_fp32_bitwise(golden):
    g = golden("fc.npz")
    for i in range(3):
        a4, b4 = g[f"fp32_{i}_a"], g[f"fp32_{i}_b"]
        mb, kb, bk, bm = a4.shape
        nb, _, bn, _ = b4.shape
        act = str(g[f"fp32_{i}_act"])
        spec = tpp.FcSpec(mb, nb, kb, bm, bn, bk, activation=tpp.UnaryKind.RELU if act == "relu" else None)
        c = tpp.alloc(tpp.TensorDesc(bm, nb * mb * bn, bm, tpp.DType.FP32))
        tpp.fc_forward(spec, to_dev(a4), to_dev(b4), c)
        assert bits(to_host(c.primary)) == bits(g[f"fp32_{i}_c"]), i


@pytest.mark.parametrize("mb,nb,kb,act", [(3, 2, 4, None), (2, 3, 2, "relu")])
def test_fc_fp32_multi_block_staged(mb, nb, kb, act):
    """FP32 fc_forward with m_b >= 2 and 64 x 64 x 64 blocks: the staged
    ordered engine with instances = m_b sharing one B per token block
    (instance stride 0 on B), bitwise vs the reference order."""
    rng = np.random.default_rng(200 + mb * 10 + nb)
    bm = bn = bk = 64
    a4 = rng.standard_normal((mb, kb, bk, bm)).astype(np.float32)
    b4 = rng.standard_normal((nb, kb, bn, bk)).astype(np.float32)
    spec = tpp.FcSpec(mb, nb, kb, bm, bn, bk, activation=tpp.UnaryKind.RELU if act else None)
    c = tpp.alloc(tpp.TensorDesc(bm, nb * mb * bn, bm, tpp.DType.FP32))
    tpp.fc_forward(spec, to_dev(a4), to_dev(b4), c)
    want = O.fc_forward_fp32(a4, b4, activation=act)
    assert bits(to_host(c.primary)) == bits(np.ascontiguousarray(want).reshape(-1))


def test_brgemm_stride_batched_shared_operand():
    """tpp_brgemm_stride_batched with inst_b = 0 (every instance reads the same
    B batch) and with both instance strides set: bitwise vs the oracle."""
    import ctypes as C
    from paper_2104_05755_b200 import _lib
    rng = np.random.default_rng(210)
    m = n = k = 64
    count, inst = 4, 3
    a = rng.standard_normal(inst * count * m * k).astype(np.float32)
    b = rng.standard_normal(inst * count * k * n).astype(np.float32)
    lib = _lib.load()
    d = tpp.GemmSpec(m, n, k, m, k, m, beta=0.0).c()
    ad, bd = to_dev(a), to_dev(b)
    for inst_b in (0, count * k * n):
        c = torch.zeros(inst * m * n, dtype=torch.float32, device="cuda")
        rc = lib.tpp_brgemm_stride_batched(C.byref(d), ad.data_ptr(), bd.data_ptr(), m * k, k * n, count,
                                           c.data_ptr(), inst, count * m * k, inst_b, m * n,
                                           _lib.stream_ptr(None))
        _lib.check(rc, "stride_batched")
        got = to_host(c).reshape(inst, n, m)
        for j in range(inst):
            ab = [O.load_a(a, j * count * m * k + i * m * k, m, k, m, "fp32") for i in range(count)]
            bb = [O.load_b(b, j * inst_b + i * k * n, k, n, k, "fp32") for i in range(count)]
            want = O.brgemm(ab, bb, np.zeros((m, n), np.float32), beta=0.0)
            assert bits(got[j].T.copy()) == bits(want), (inst_b, j)


def test_layernorm_blocked_bitwise():
    rng = np.random.default_rng(21)
    # (4,16,32,64) and (700,1,32,64) take the TMA pipeline (the latter wraps
    # each CTA's buffer ring several times); the others the generic kernels
    for (n_b, m_b, bn, bm, dt) in ((4, 16, 32, 64, "bf16"), (2, 3, 48, 32, "fp32"), (3, 2, 8, 64, "bf16"),
                                   (700, 1, 32, 64, "bf16"), (5, 5, 48, 64, "bf16")):
        x = rng.normal(0, 1, (n_b, m_b, bn, bm)).astype(np.float32) + 0.3
        if dt == "bf16":
            x = O.fp32_to_bf16_rne(x)
        gam = (1 + 0.1 * rng.standard_normal(m_b * bm)).astype(np.float32)
        bet = (0.1 * rng.standard_normal(m_b * bm)).astype(np.float32)
        mean = torch.empty(n_b * bn, dtype=torch.float32, device="cuda")
        var = torch.empty_like(mean)
        out = tpp.layernorm_blocked(to_dev(x), n_b, m_b, bn, bm, 1e-5, to_dev(gam), to_dev(bet),
                                    mean_out=mean, var_out=var)
        xf = O.bf16_to_fp32(x) if dt == "bf16" else x
        logical = xf.transpose(0, 2, 1, 3).reshape(n_b * bn, m_b * bm)  # tokens x features
        ref, mu, vr = O.layernorm(logical, gam[None, :], bet[None, :], 1e-5)
        ref = ref.reshape(n_b, bn, m_b, bm).transpose(0, 2, 1, 3)
        if dt == "bf16":
            assert np.array_equal(to_host(out), O.fp32_to_bf16_rne(ref).reshape(-1))
        else:
            assert bits(to_host(out)) == bits(ref.reshape(-1))
        assert bits(to_host(mean)) == bits(mu.astype(np.float32))
        assert bits(to_host(var)) == bits(vr.astype(np.float32))


# ---------------------------------------------------------------------------
# BF16 tensor-core layers (tcgen05): normwise tolerance vs the oracle
# ---------------------------------------------------------------------------

def _fc_case(rng, Nb, Cb, bn, bc, Kb, bk, act, bias=True, residual=False, block_n=0,
             mask=False, nb_sel=None):
    x = O.fp32_to_bf16_rne(rng.normal(0, 1, (Nb, Cb, bn, bc)).astype(np.float32))
    wv = vnni_weights(rng, Kb, Cb, bk, bc, 0.05)
    b = O.fp32_to_bf16_rne(rng.normal(0, 0.5, Kb * bk).astype(np.float32)) if bias else None
    res = O.fp32_to_bf16_rne(rng.normal(0, 1, (Nb, Kb, bn, bk)).astype(np.float32)) if residual else None
    layer = tpp.FcLayer(Kb, Cb, bk, bc, to_dev(wv), bias=to_dev(b) if bias else None,
                        activation={"relu": tpp.UnaryKind.RELU, "gelu": tpp.UnaryKind.GELU, None: None}[act],
                        block_n=block_n)
    mbuf = torch.zeros(Nb * Kb * bn * (bk // 8), dtype=torch.uint8, device="cuda") if mask else None
    out = layer.forward(to_dev(x), Nb, bn, residual=to_dev(res) if residual else None, relu_mask=mbuf)
    got_bits = to_host(out).reshape(Nb, Kb, bn, bk)
    sel = list(range(Nb)) if nb_sel is None else list(nb_sel)
    want_bits, want_mask, _ = O.fc_forward_bf16(x, wv, b, activation=act, residual_bits=res, nb_sel=sel)
    got = bf16_bits_to_f32(got_bits[sel])
    want = O.bf16_to_fp32(want_bits)
    err = normwise(got, want)
    exact = float(np.mean(got_bits[sel] == want_bits))
    mask_agree = None
    if mask:
        mb_host = to_host(mbuf).reshape(Nb, Kb, bn, bk // 8)[sel]
        got_mask = np.unpackbits(mb_host, axis=-1, bitorder="little").astype(bool)
        mask_agree = float(np.mean(got_mask == want_mask))
    return err, exact, mask_agree


@pytest.mark.parametrize("block_n", [64, 128, 256])
def test_fc_bf16_relu_bias_tile_widths(block_n):
    rng = np.random.default_rng(30)
    err, exact, mask_agree = _fc_case(rng, 4, 4, 64, 64, 4, 64, "relu", block_n=block_n, mask=True)
    assert err <= BF16_TOL, err
    assert exact > 0.9, exact
    assert mask_agree > 0.999, mask_agree


def test_fc_bf16_golden(golden):
    g = golden("fc.npz")
    i = 2  # the TC-compatible golden case: bc = bk = 64, bn = 32
    x, wv, bias = g[f"bf16_{i}_x"], g[f"bf16_{i}_w"], g[f"bf16_{i}_bias"]
    Nb, Cb, bn, bc = x.shape
    Kb, _, _, bk, _ = wv.shape
    layer = tpp.FcLayer(Kb, Cb, bk, bc, to_dev(wv), bias=to_dev(bias), activation=tpp.UnaryKind.RELU)
    out = layer.forward(to_dev(x), Nb, bn)
    got = to_host(out).reshape(Nb, Kb, bn, bk)
    want = g[f"bf16_{i}_out"]
    assert normwise(bf16_bits_to_f32(got), O.bf16_to_fp32(want)) <= BF16_TOL


def test_fc_bf16_gelu_residual_bn32():
    rng = np.random.default_rng(31)
    err, exact, _ = _fc_case(rng, 8, 3, 32, 64, 3, 64, "gelu", residual=True)
    assert err <= BF16_TOL, err
    assert exact > 0.9, exact


def test_fc_bf16_cfg2_full():
    """BASELINE cfg 2 (N=C=K=1024, bias+ReLU) at full size; the oracle checks
    sampled token blocks exactly as the reference would compute them."""
    rng = np.random.default_rng(0)
    err, exact, _ = _fc_case(rng, 16, 16, 64, 64, 16, 64, "relu", nb_sel=[0, 7, 15])
    assert err <= BF16_TOL, err
    assert exact > 0.9, exact


def test_fc_bf16_cfg3_shapes_sampled():
    """BASELINE cfg 3 FC1 (1024->4096, GELU) and FC2 (4096->1024 + residual)
    at their real K / N, tokens sampled (bn = 32)."""
    rng = np.random.default_rng(1)
    err, _, _ = _fc_case(rng, 8, 16, 32, 64, 64, 64, "gelu", bias=False, nb_sel=[0, 5])
    assert err <= BF16_TOL, err
    err, _, _ = _fc_case(rng, 4, 64, 32, 64, 16, 64, None, bias=False, residual=True, nb_sel=[1, 3])
    assert err <= BF16_TOL, err


def test_fc_bf16_ragged_tokens():
    """Token count not a multiple of the 128-row tile (TMA zero-fill + masked stores)."""
    rng = np.random.default_rng(32)
    err, _, _ = _fc_case(rng, 3, 2, 32, 64, 2, 64, "relu")  # 96 tokens
    assert err <= BF16_TOL, err
    err, _, _ = _fc_case(rng, 5, 2, 64, 64, 4, 64, None)    # 320 tokens
    assert err <= BF16_TOL, err


def _conv_case(rng, N, Cb, Kb, H, W, n_sel=None):
    x = O.fp32_to_bf16_rne(rng.random((N, Cb, H, W, 64)).astype(np.float32))
    wl = O.fp32_to_bf16_rne(rng.normal(0, np.sqrt(2 / (9 * 64 * Cb)), (Kb, Cb, 3, 3, 64, 64)).astype(np.float32))
    wv = wl.reshape(Kb, Cb, 3, 3, 64, 32, 2).transpose(0, 1, 2, 3, 5, 4, 6).copy()
    spec = tpp.ConvSpec(N, Cb, Kb, H, W)
    conv = tpp.Conv2d(spec, to_dev(wv))
    out = conv.forward(to_dev(x))
    sel = list(range(N)) if n_sel is None else n_sel
    got = bf16_bits_to_f32(to_host(out).reshape(N, Kb, H, W, 64)[sel])
    want_bits, _ = O.conv2d_fwd_bf16(x, wv, n_sel=sel)
    err_f = normwise(got, O.bf16_to_fp32(want_bits))
    # backward data: dI = conv(dO, flip(W)^T)
    dout = O.fp32_to_bf16_rne(rng.normal(0, 1, (N, Kb, H, W, 64)).astype(np.float32))
    din = conv.backward_data(to_dev(dout))
    got_b = bf16_bits_to_f32(to_host(din).reshape(N, Cb, H, W, 64)[sel])
    wbwd = O.conv_weights_bwd_data(wv)
    want_b, _ = O.conv2d_fwd_bf16(dout, wbwd, n_sel=sel)
    err_b = normwise(got_b, O.bf16_to_fp32(want_b))
    return err_f, err_b


def test_conv_small_fwd_bwd():
    rng = np.random.default_rng(40)
    err_f, err_b = _conv_case(rng, 2, 1, 1, 9, 12)
    assert err_f <= BF16_TOL and err_b <= BF16_TOL, (err_f, err_b)
    err_f, err_b = _conv_case(rng, 1, 2, 2, 6, 64)
    assert err_f <= BF16_TOL and err_b <= BF16_TOL, (err_f, err_b)


def test_conv_golden(golden):
    """Reference offset-BRGEMM conv fixture is 8-channel; check the oracle
    composition the GPU test relies on matches it (pinning), then the GPU
    conv on the cfg-4 image shape against that oracle."""
    g = golden("conv.npz")
    out, _ = O.conv2d_fwd_bf16(g["x"], g["w"])
    assert np.array_equal(out, g["out"])
    rng = np.random.default_rng(41)
    err_f, err_b = _conv_case(rng, 2, 1, 1, 56, 56, n_sel=[1])
    assert err_f <= BF16_TOL and err_b <= BF16_TOL, (err_f, err_b)


def test_conv_multi_wave_shapes():
    """More than one wave of 2-row tiles (persistent CTAs walk several tiles and
    reuse their accumulator / halo rings), odd and even tile counts per image,
    ragged widths."""
    rng = np.random.default_rng(42)
    err_f, err_b = _conv_case(rng, 6, 1, 1, 56, 56, n_sel=[0, 3, 5])   # 168 tiles, 28 per image: pairs
    assert err_f <= BF16_TOL and err_b <= BF16_TOL, (err_f, err_b)
    err_f, err_b = _conv_case(rng, 12, 1, 1, 26, 40, n_sel=[0, 11])   # 13 tiles per image: single CTAs
    assert err_f <= BF16_TOL and err_b <= BF16_TOL, (err_f, err_b)
    err_f, err_b = _conv_case(rng, 12, 1, 1, 28, 20, n_sel=[4, 7])    # 14 per image, ragged width: pairs
    assert err_f <= BF16_TOL and err_b <= BF16_TOL, (err_f, err_b)
    # W = 64 (the widest tile row), a one-row image, a 2-pixel-wide image
    for n, h, w in ((2, 7, 64), (3, 1, 5), (2, 9, 2)):
        err_f, err_b = _conv_case(rng, n, 1, 1, h, w)
        assert err_f <= BF16_TOL and err_b <= BF16_TOL, (n, h, w, err_f, err_b)


def _conv_generic_case(rng, N, Cb, Kb, H, W, R, S, pad, stride):
    """Shapes outside the fused halo kernels: the reference composition (padded
    input, OFFSET BRGEMM over the (r, s, cb) taps per output row) on the
    grouped tcgen05 BRGEMM; forward against the oracle composition, backward-
    data against an FP64 restatement of the adjoint."""
    from paper_2104_05755_b200 import _lib
    x = O.fp32_to_bf16_rne(rng.random((N, Cb, H, W, 64)).astype(np.float32))
    wl = O.fp32_to_bf16_rne(rng.normal(0, np.sqrt(2 / (R * S * 64 * Cb)), (Kb, Cb, R, S, 64, 64)).astype(np.float32))
    wv = wl.reshape(Kb, Cb, R, S, 64, 32, 2).transpose(0, 1, 2, 3, 5, 4, 6).copy()
    spec = tpp.ConvSpec(N, Cb, Kb, H, W, r=R, s=S, pad=pad, stride=stride)
    assert not spec.fused
    conv = tpp.Conv2d(spec, to_dev(wv))
    out = conv.forward(to_dev(x))
    torch.cuda.synchronize()
    assert _lib.last_config().startswith("brgemm_grouped_kernel"), _lib.last_config()
    P, Q = spec.p, spec.q
    got = bf16_bits_to_f32(to_host(out).reshape(N, Kb, P, Q, 64))
    want_bits, _ = O.conv2d_fwd_bf16(x, wv, pad=pad, stride=stride)
    assert want_bits.shape == (N, Kb, P, Q, 64)
    err_f = normwise(got, O.bf16_to_fp32(want_bits))
    dout = O.fp32_to_bf16_rne(rng.normal(0, 1, (N, Kb, P, Q, 64)).astype(np.float32))
    din = conv.backward_data(to_dev(dout))
    got_b = bf16_bits_to_f32(to_host(din).reshape(N, Cb, H, W, 64))
    err_b = normwise(got_b, O.conv2d_bwd_data_fp64(dout, wv, H, W, pad, stride))
    return err_f, err_b


@pytest.mark.parametrize("N,Cb,Kb,H,W,R,S,pad,stride", [
    (2, 1, 1, 9, 11, 3, 3, 1, 2),     # ResNet 3x3 stride-2 downsampling
    (1, 2, 2, 8, 8, 1, 1, 0, 2),      # 1x1 stride-2 projection shortcut
    (1, 1, 2, 13, 13, 7, 7, 3, 2),    # the 7x7 stride-2 stem
    (1, 1, 1, 5, 70, 3, 3, 1, 1),     # W > 64
    (2, 2, 1, 6, 7, 3, 3, 0, 1),      # 'valid' padding
])
def test_conv_generic_shapes(N, Cb, Kb, H, W, R, S, pad, stride):
    rng = np.random.default_rng(43 + R + stride)
    err_f, err_b = _conv_generic_case(rng, N, Cb, Kb, H, W, R, S, pad, stride)
    assert err_f <= BF16_TOL and err_b <= BF16_TOL, (err_f, err_b)


# ---------------------------------------------------------------------------
# 1-D dilated conv (kernels.py:336-378): stride BRGEMM over taps, bitwise
# ---------------------------------------------------------------------------

def test_dilated_conv1d_bitwise(golden):
    g = golden("dilated.npz")
    for name in ("small", "atac"):
        c, k, s, d, w, q = (int(v) for v in g[f"{name}_shape"])
        x = tpp.from_array(g[f"{name}_x"], device="cuda")
        wt = tpp.from_array(g[f"{name}_w"], device="cuda")
        out = tpp.alloc(tpp.TensorDesc(k, q, k, tpp.DType.FP32), device="cuda")
        tpp.dilated_conv1d_forward(tpp.DilatedConvSpec(c, k, w, q, s, d), x, wt, out)
        assert bits(tpp.to_array(out)) == bits(g[f"{name}_out"]), name


def test_dilated_conv1d_impulse_and_guard():
    """test_kernels.py:395-409 and 423-425: an impulse reproduces the taps."""
    c_, k_, s_, d_, q_ = 1, 2, 3, 2, 6
    w_ = q_ + (s_ - 1) * d_
    x = np.zeros((c_, w_), dtype=np.float32)
    x[0, 4] = 1.0
    wt = np.arange(s_ * c_ * k_, dtype=np.float32).reshape(s_ * c_, k_) + 1
    out = tpp.alloc(tpp.TensorDesc(k_, q_, k_, tpp.DType.FP32), device="cuda")
    tpp.dilated_conv1d_forward(tpp.DilatedConvSpec(c_, k_, w_, q_, s_, d_), tpp.from_array(x, device="cuda"),
                               tpp.from_array(wt, device="cuda"), out)
    o = tpp.to_array(out)
    for k2 in range(k_):
        for qq in range(q_):
            hits = [wt[s2, k2] for s2 in range(s_) if qq + s2 * d_ == 4]
            assert o[k2, qq] == (hits[0] if hits else 0.0)
    with pytest.raises(tpp.TensorError):
        tpp.DilatedConvSpec(1, 1, 10, 9, 3, 2)


# ---------------------------------------------------------------------------
# dense fast paths (eltwise_fast.cu) == the generic kernels, bit for bit
# ---------------------------------------------------------------------------

def _padded(x: np.ndarray, dt, pad: int):
    """Column-major view of x with ld = rows + pad (pad 0: the dense fast path)."""
    m, n = x.shape
    ld = m + pad
    buf = np.zeros((ld, n), dtype=np.float32)
    buf[:m] = x
    flat = torch.from_numpy(np.asfortranarray(buf).reshape(-1, order="F").copy()).cuda()
    if dt is tpp.DType.BF16:
        flat = tpp.convert(tpp.TensorView(tpp.TensorDesc(ld, n, ld, tpp.DType.FP32), flat), tpp.DType.BF16).primary
    return tpp.TensorView(tpp.TensorDesc(m, n, ld, dt), flat)


def _dense_bits(v):
    """Bit patterns of the logical window, NaN payloads canonicalised (the
    generic kernels' compiled ReLU may canonicalise a NaN; the reference and
    the fast path keep the operand's payload)."""
    m, n, ld = v.desc.rows, v.desc.cols, v.desc.ld
    a = np.ascontiguousarray(to_host(v.primary).reshape(n, ld)[:, :m])
    if a.dtype == np.uint16:
        a = a.copy()
        a[((a & 0x7F80) == 0x7F80) & ((a & 0x7F) != 0)] = 0x7FC0
        return a.tobytes()
    return bits(a)


def test_dense_fast_paths_match_generic():
    rng = np.random.default_rng(77)
    m, n = 256, 96
    x = rng.standard_normal((m, n)).astype(np.float32) * 3
    x.flat[::97] = np.nan
    x.flat[5::101] = -0.0
    x.flat[7::103] = np.inf
    y = rng.standard_normal((m, n)).astype(np.float32)
    z = rng.standard_normal((m, n)).astype(np.float32)
    U = tpp.UnaryKind
    for dt in (tpp.DType.FP32, tpp.DType.BF16):
        for odt in (tpp.DType.FP32, tpp.DType.BF16):
            res = {}
            for pad in (0, 8):
                xv, yv, zv = _padded(x, dt, pad), _padded(y, dt, pad), _padded(z, dt, pad)
                outs = {}
                for kind in (U.IDENTITY, U.SQUARE, U.INC, U.SQRT, U.RECIPROCAL, U.RSQRT, U.EXP, U.RELU, U.GELU):
                    o = tpp.TensorView(tpp.TensorDesc(m, n, m + pad, odt),
                                       torch.zeros((m + pad) * n, dtype=odt.storage, device="cuda"))
                    tpp.apply_unary(kind, xv, o, bitmask_output=kind is U.RELU)
                    outs[kind] = _dense_bits(o)
                    if kind is U.RELU:
                        outs["mask"] = to_host(o.secondary).tolist() if pad == 0 else None
                for kind in (tpp.BinaryKind.ADD, tpp.BinaryKind.MUL, tpp.BinaryKind.DIV, tpp.BinaryKind.MAX):
                    o = tpp.TensorView(tpp.TensorDesc(m, n, m + pad, odt),
                                       torch.zeros((m + pad) * n, dtype=odt.storage, device="cuda"))
                    tpp.apply_binary(kind, xv, yv, o)
                    outs[kind] = _dense_bits(o)
                o = tpp.TensorView(tpp.TensorDesc(m, n, m + pad, odt),
                                   torch.zeros((m + pad) * n, dtype=odt.storage, device="cuda"))
                tpp.apply_ternary(tpp.TernaryKind.MULADD, xv, yv, zv, o)
                outs["muladd"] = _dense_bits(o)
                res[pad] = outs
            for k in res[0]:
                if k == "mask":
                    continue
                assert res[0][k] == res[8][k], (dt, odt, k)
    # transforms: fast (aligned, even) vs the oracle's index formulas
    a = rng.integers(0, 1 << 16, size=(64, 48), dtype=np.uint16)
    av = tpp.TensorView(tpp.TensorDesc(64, 48, 64, tpp.DType.BF16),
                        torch.from_numpy(a.reshape(-1, order="F").view(np.int16).copy()).cuda().view(torch.bfloat16))
    t = tpp.alloc(tpp.TensorDesc(48, 64, 48, tpp.DType.BF16))
    tpp.transform(av, tpp.TransformSpec(tpp.TransformKind.TRANSPOSE), t)
    assert np.array_equal(tpp.bits_of(t), a.T)
    # full 64x64 tiles: the 16-byte-access transpose (incl. a padded output ld)
    for (rr, cc, old) in ((128, 192, 192), (192, 64, 72)):
        b = rng.integers(0, 1 << 16, size=(rr, cc), dtype=np.uint16)
        bv = tpp.TensorView(tpp.TensorDesc(rr, cc, rr, tpp.DType.BF16),
                            torch.from_numpy(b.reshape(-1, order="F").view(np.int16).copy()).cuda().view(torch.bfloat16))
        tb = tpp.TensorView(tpp.TensorDesc(cc, rr, old, tpp.DType.BF16),
                            torch.zeros(old * rr, dtype=torch.bfloat16, device="cuda"))
        tpp.transform(bv, tpp.TransformSpec(tpp.TransformKind.TRANSPOSE), tb)
        assert np.array_equal(tpp.bits_of(tb), b.T), (rr, cc, old)
    vn = tpp.alloc(tpp.TensorDesc(128, 24, 128, tpp.DType.BF16))
    tpp.transform(av, tpp.TransformSpec(tpp.TransformKind.VNNI, alpha=2), vn)
    got = tpp.bits_of(vn)
    for g_ in range(24):
        for mm in range(64):
            assert got[2 * mm, g_] == a[mm, 2 * g_] and got[2 * mm + 1, g_] == a[mm, 2 * g_ + 1]
    vt = tpp.alloc(tpp.TensorDesc(96, 32, 96, tpp.DType.BF16))
    tpp.transform(vn, tpp.TransformSpec(tpp.TransformKind.VNNI_TO_VNNIT, alpha=2, alpha_out=2, rows=64, cols=48), vt)
    gt = tpp.bits_of(vt)
    for h in range(32):
        for kk in range(48):
            assert gt[2 * kk, h] == a[2 * h, kk] and gt[2 * kk + 1, h] == a[2 * h + 1, kk]


# ---------------------------------------------------------------------------
# conv backward-weights: normwise vs the float64 composition
# ---------------------------------------------------------------------------

def _conv_dw_case(rng, N, Cb, Kb, H, W):
    spec = tpp.ConvSpec(N, Cb, Kb, H, W)
    x = O.fp32_to_bf16_rne(rng.uniform(0, 1, (N, Cb, H, W, 64)).astype(np.float32))
    do = O.fp32_to_bf16_rne(rng.standard_normal((N, Kb, H, W, 64)).astype(np.float32))
    wv = to_dev(O.fp32_to_bf16_rne(rng.standard_normal(Kb * Cb * 9 * 64 * 64).astype(np.float32) * 0.1))
    conv = tpp.Conv2d(spec, wv)
    dw = conv.backward_weights(to_dev(x), to_dev(do))
    got = to_host(dw).reshape(Kb, Cb, 3, 3, 64, 64).astype(np.float64)
    want = O.conv2d_bwd_weights(x, do)
    return normwise(got, want)


def test_conv_backward_weights():
    rng = np.random.default_rng(55)
    assert _conv_dw_case(rng, 2, 1, 1, 9, 12) <= 1e-5
    assert _conv_dw_case(rng, 3, 2, 2, 7, 20) <= 1e-5
    assert _conv_dw_case(rng, 4, 1, 1, 56, 56) <= 1e-5


def test_layernorm_blocked_tolerance_mode():
    """exact=False (tree-ordered sums, FMA scaling): statistics within 1e-5
    relative, outputs within the BF16 tolerance and nearly all bit-identical."""
    rng = np.random.default_rng(23)
    n_b, m_b, bn, bm = 40, 16, 32, 64
    x = O.fp32_to_bf16_rne(rng.normal(0, 1, (n_b, m_b, bn, bm)).astype(np.float32) + 0.3)
    gam = (1 + 0.1 * rng.standard_normal(m_b * bm)).astype(np.float32)
    bet = (0.1 * rng.standard_normal(m_b * bm)).astype(np.float32)
    res = {}
    for exact in (True, False):
        mean = torch.empty(n_b * bn, dtype=torch.float32, device="cuda")
        var = torch.empty_like(mean)
        out = tpp.layernorm_blocked(to_dev(x), n_b, m_b, bn, bm, 1e-5, to_dev(gam), to_dev(bet),
                                    mean_out=mean, var_out=var, exact=exact)
        res[exact] = (to_host(out), to_host(mean), to_host(var))
    (oe, me, ve), (of, mf, vf) = res[True], res[False]
    assert normwise(mf, me) <= 1e-5 and normwise(vf, ve) <= 1e-5
    assert normwise(bf16_bits_to_f32(of), bf16_bits_to_f32(oe)) <= BF16_TOL
    assert np.mean(of == oe) > 0.95


# ---------------------------------------------------------------------------
# PRNG / DROPOUT / DROPOUT_INV (ops.py:195-236, 378-382, 430-444): bitwise
# ---------------------------------------------------------------------------

def _words(st):
    return st.words().cpu().numpy().astype(np.uint32)


def test_prng_seed_and_fill_bitwise(golden):
    g = golden("prng.npz")
    for s, want in zip(g["seeds"], g["seed_words"]):
        assert np.array_equal(_words(tpp.PrngState(int(s), 8)), want)
    src = tpp.alloc(tpp.TensorDesc(1, 1, 1, tpp.DType.FP32))
    st = tpp.PrngState(123, 6)
    src.tertiary = {"prng": st}
    f1 = tpp.alloc(tpp.TensorDesc(64, 6, 64, tpp.DType.FP32))
    tpp.apply_unary(tpp.UnaryKind.PRNG, src, f1)
    assert bits(to_host(f1.primary)) == bits(g["fill1"])
    f2 = tpp.alloc(tpp.TensorDesc(37, 6, 40, tpp.DType.FP32))
    tpp.apply_unary(tpp.UnaryKind.PRNG, src, f2)
    got = O.strided2d(to_host(f2.primary), 0, 37, 6, 40)
    assert bits(got) == bits(O.strided2d(g["fill2"], 0, 37, 6, 40))
    assert np.array_equal(_words(st), g["state_after"])
    # 70001 rows: 1094 row segments reached through the GF(2) jump tables
    lst = tpp.PrngState(99, 3)
    lsrc = tpp.alloc(tpp.TensorDesc(1, 1, 1, tpp.DType.FP32))
    lsrc.tertiary = {"prng": lst}
    n = int(g["long_rows"])
    lf = tpp.alloc(tpp.TensorDesc(n, 3, n, tpp.DType.FP32))
    tpp.apply_unary(tpp.UnaryKind.PRNG, lsrc, lf)
    assert bits(tpp.to_array(lf)[g["long_idx"]]) == bits(g["long_sample"])
    assert np.array_equal(_words(lst), g["long_state"])


def test_dropout_bitwise(golden):
    g = golden("prng.npz")
    x = g["x"]
    m, n = x.shape
    xv = tpp.from_array(x)
    xv.tertiary = {"prng": tpp.PrngState(7, n)}
    d1 = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.FP32))
    tpp.apply_unary(tpp.UnaryKind.DROPOUT, xv, d1, dropout_p=0.3)
    d2 = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.FP32))
    tpp.apply_unary(tpp.UnaryKind.DROPOUT, xv, d2, dropout_p=0.3)
    assert bits(to_host(d1.primary)) == bits(g["d1"]) and bits(to_host(d2.primary)) == bits(g["d2"])
    assert np.array_equal(to_host(d1.secondary), g["m1"])
    assert np.array_equal(to_host(d2.secondary), g["m2"])
    dyv = tpp.from_array(g["dy"])
    dyv.secondary = d1.secondary
    di = tpp.alloc(d1.desc)
    tpp.apply_unary(tpp.UnaryKind.DROPOUT_INV, dyv, di, dropout_p=0.3)
    assert bits(to_host(di.primary)) == bits(g["dinv"])
    tpp.apply_unary(tpp.UnaryKind.DROPOUT_INV, dyv, di, dropout_p=1.0)
    assert bits(to_host(di.primary)) == bits(g["dinv_p1"])
    xb = tpp.from_array(x, tpp.DType.BF16)
    wrong = tpp.PrngState(5, 4)
    xb.tertiary = {"prng": wrong}
    db = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.BF16))
    tpp.apply_unary(tpp.UnaryKind.DROPOUT, xb, db, dropout_p=0.1)
    assert bf16_equal(to_host(db.primary), g["db"])
    assert np.array_equal(to_host(db.secondary), g["mb"])
    assert np.array_equal(_words(wrong), g["wrong_after"])


@pytest.mark.parametrize("rows,cols,ld,p,dt", [
    (4096, 1024, 4096, 0.1, "fp32"),    # full-size activation block
    (1000, 77, 1003, 0.5, "fp32"),      # ragged tile edges, padded ld
    (513, 33, 513, 0.9, "bf16"),
    (130, 5, 130, 0.25, "fp64"),
    (64, 3, 64, 0.99999999, "fp32"),    # float32(p) == 1.0: nothing kept
    (4100, 40, 4100, 0.0, "bf16"),      # p = 0: everything kept, scale 1
    # TMA-fed fused kernel (rows % 64 == 0): two interleaved streams per lane
    (8192, 1024, 8192, 0.1, "bf16"),    # 2 + 2 slabs per warp
    (1984, 45, 2000, 0.3, "bf16"),      # last warp: stream A only; ragged columns, padded ld
    (4096, 70, 4104, 0.5, "fp32"),
    (640, 33, 640, 0.2, "fp32"),
    (16384, 8, 16384, 0.1, "bf16"),     # one column group, many warps
    (16384, 2048, 16384, 0.1, "bf16"),  # TMA fused: 4 + 4 slabs per warp, stream B one level-2 jump
])
def test_dropout_matches_oracle(rows, cols, ld, p, dt):
    rng = np.random.default_rng(rows + cols)
    x = rng.standard_normal((rows, cols))
    if dt == "fp32":
        x = x.astype(np.float32)
    dtype = {"fp32": tpp.DType.FP32, "bf16": tpp.DType.BF16, "fp64": tpp.DType.FP64}[dt]
    buf = np.zeros(ld * (cols - 1) + rows, dtype=np.float64 if dt == "fp64" else np.float32)
    for j in range(cols):
        buf[j * ld: j * ld + rows] = x[:, j]
    desc = tpp.TensorDesc(rows, cols, ld, dtype)
    if dt == "bf16":
        xv = tpp.from_array(x.astype(np.float32), dtype)
        xw = O.bf16_to_fp32(tpp.bits_of(xv))
    else:
        xv = tpp.TensorView(desc, to_dev(buf))
        xw = x
    xv.tertiary = {"prng": tpp.PrngState(2024, cols)}
    out = tpp.alloc(tpp.TensorDesc(rows, cols, rows, dtype))
    tpp.apply_unary(tpp.UnaryKind.DROPOUT, xv, out, dropout_p=p)
    want, keep = O.dropout(xw, O.prng_seed(2024, cols), p)
    assert np.array_equal(to_host(out.secondary), O.bool_to_mask(keep))
    if dt == "bf16":
        assert np.array_equal(tpp.bits_of(out), O.fp32_to_bf16_rne(want))
    else:
        assert bits(tpp.to_array(out)) == bits(want)


def test_dropout_statistics_and_errors():
    """verify.check_dropout: keep rate within 3 sigma of 1-p over 10^6 draws,
    kept values exactly 1/(1-p); InvalidSpecError without a state or p out of
    range (test_ops.py:526-556)."""
    m = n = 1000
    ones = np.ones((m, n), dtype=np.float32)
    for p in (0.1, 0.5, 0.9):
        v = tpp.from_array(ones)
        v.tertiary = {"prng": tpp.PrngState(2024, n)}
        out = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.FP32))
        tpp.apply_unary(tpp.UnaryKind.DROPOUT, v, out, dropout_p=p)
        keep = tpp.mask_to_bool(out.secondary, m, n)
        vals = tpp.to_array(out)
        sigma = (p * (1 - p) / (m * n)) ** 0.5
        assert abs(keep.mean() - (1 - p)) <= 3 * sigma
        assert np.all(vals[~keep] == 0)
        assert np.all(vals[keep] == np.float32(1 / (1 - p)))
    x = tpp.from_array(np.ones((2, 2), dtype=np.float32))
    out = tpp.alloc(tpp.TensorDesc(2, 2, 2, tpp.DType.FP32))
    with pytest.raises(tpp.InvalidSpecError):
        tpp.apply_unary(tpp.UnaryKind.DROPOUT, x, out, dropout_p=0.5)
    x.tertiary = {"prng": tpp.PrngState(0, 2)}
    with pytest.raises(tpp.InvalidSpecError):
        tpp.apply_unary(tpp.UnaryKind.DROPOUT, x, out, dropout_p=1.5)
    tpp.apply_unary(tpp.UnaryKind.DROPOUT, x, out, dropout_p=0.0)
    assert np.all(tpp.to_array(out) == 1.0)


# ---------------------------------------------------------------------------
# QUANTIZE / DEQUANTIZE (ops.py:447-469): bitwise
# ---------------------------------------------------------------------------

def test_quantize_dequantize_bitwise(golden):
    g = golden("quant.npz")
    for name in ("uniform", "normal", "nan", "zeros", "ties"):
        x = g[name + "_x"]
        m, n = x.shape
        q = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.INT8))
        tpp.apply_unary(tpp.UnaryKind.QUANTIZE, tpp.from_array(x), q)
        assert q.tertiary["scale"] == float(g[name + "_scale"]), name
        assert np.array_equal(to_host(q.primary), g[name + "_q"]), name
        d = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.FP32))
        tpp.apply_unary(tpp.UnaryKind.DEQUANTIZE, q, d)
        assert bits(to_host(d.primary)) == bits(g[name + "_d"]), name
    xv = tpp.from_array(g["normal_x"])
    xv.tertiary = {"scale": 0.01}
    q = tpp.alloc(tpp.TensorDesc(37, 29, 37, tpp.DType.INT8))
    tpp.apply_unary(tpp.UnaryKind.QUANTIZE, xv, q)
    assert np.array_equal(to_host(q.primary), g["given_q"])


def test_quantize_full_size_matches_oracle():
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((2048, 1536)) * 4).astype(np.float32)
    q = tpp.alloc(tpp.TensorDesc(2048, 1536, 2048, tpp.DType.INT8))
    tpp.apply_unary(tpp.UnaryKind.QUANTIZE, tpp.from_array(x), q)
    want, scale = O.quantize(x)
    assert q.tertiary["scale"] == scale
    assert np.array_equal(tpp.to_array(q), want)
    with pytest.raises(tpp.InvalidSpecError):
        tpp.apply_unary(tpp.UnaryKind.DEQUANTIZE, tpp.from_array(np.zeros((2, 2), np.int8)),
                        tpp.alloc(tpp.TensorDesc(2, 2, 2, tpp.DType.FP32)))


# ---------------------------------------------------------------------------
# INT8 BRGEMM on tcgen05 kind::i8 (contraction.py:75-85, 184-189): integer
# sums are order-independent, so the tensor engine must equal the reference
# bit for bit (including int32 wrap-around)
# ---------------------------------------------------------------------------

def _int8_ref(a_list, b_list, c0, beta):
    """Modular int32 reference: int64 sums wrapped to int32 == numpy's
    wrapping int32 accumulation in any order."""
    acc = np.zeros(c0.shape, dtype=np.int64)
    for a, b in zip(a_list, b_list):  # |partial| < 2^53: float64 BLAS is exact here
        acc += (a.astype(np.float64) @ b.astype(np.float64)).astype(np.int64)
    if beta == 0.0:
        base = np.zeros(c0.shape, np.int64)
    else:
        base = c0.astype(np.int64) * (1 if beta == 1.0 else int(np.int32(beta)))
    return ((base + acc) & 0xFFFFFFFF).astype(np.uint32).view(np.int32)


@pytest.mark.parametrize("m,n,k,count,beta,engine", [
    (64, 64, 64, 16, 1.0, "tensor"),       # cfg 1 shape: sliced reduction + red.add
    (300, 200, 520, 3, 0.0, "tensor"),     # ragged M/N/K tiles (TMA zero fill)
    (1024, 1024, 1024, 4, 1.0, "auto"),    # full tiles, BN 256
    (128, 96, 4096, 1, 0.5, "tensor"),     # beta 0.5 -> int32(0) (truncation)
    (256, 48, 384, 5, -2.7, "tensor"),     # beta -2.7 -> -2, BN 64
    (4096, 2048, 256, 2, 1.0, "auto"),     # a full wave of CTA pairs (cta_group::2)
    (4000, 2000, 200, 1, 0.0, "tensor"),   # pairs with ragged M / N / K edges
])
def test_int8_tensor_engine_exact(m, n, k, count, beta, engine):
    rng = np.random.default_rng(m + n + k)
    lda = -(-m // 16) * 16
    ldb = -(-k // 16) * 16
    a_l = [rng.integers(-128, 128, (m, k), dtype=np.int8) for _ in range(count)]
    b_l = [rng.integers(-128, 128, (k, n), dtype=np.int8) for _ in range(count)]
    abuf = np.zeros((count, k, lda), np.int8)
    bbuf = np.zeros((count, n, ldb), np.int8)
    for i in range(count):
        abuf[i, :, :m] = a_l[i].T
        bbuf[i, :, :k] = b_l[i].T
    c0 = rng.integers(-1000, 1000, (m, n), dtype=np.int32)
    c = tpp.from_array(c0)
    eng = tpp.Engine.TENSOR if engine == "tensor" else tpp.Engine.AUTO
    spec = tpp.GemmSpec(m, n, k, lda, ldb, m, in_dtype=tpp.DType.INT8, out_dtype=tpp.DType.INT32,
                        beta=beta, engine=eng)
    tpp.brgemm(spec, tpp.BrgemmBatch.stride(to_dev(abuf.reshape(-1)), to_dev(bbuf.reshape(-1)),
                                            k * lda, n * ldb, count), c)
    want = _int8_ref(a_l, b_l, c0, beta)
    assert np.array_equal(tpp.to_array(c), want)
    if m * n * k * count <= 64 * 64 * 64 * 16:  # the reference's own ordered loop, small case
        c2 = tpp.from_array(c0)
        spec2 = tpp.GemmSpec(m, n, k, lda, ldb, m, in_dtype=tpp.DType.INT8, out_dtype=tpp.DType.INT32,
                             beta=beta, engine=tpp.Engine.ORDERED)
        tpp.brgemm(spec2, tpp.BrgemmBatch.stride(to_dev(abuf.reshape(-1)), to_dev(bbuf.reshape(-1)),
                                                 k * lda, n * ldb, count), c2)
        assert np.array_equal(tpp.to_array(c2), want)


def test_int8_tensor_engine_wraps_and_saturation_free():
    """127*127*K beyond 2^31 wraps exactly like numpy int32 (no saturation);
    and the reference's 127^2 * 300 known answer (test_gemm.py:245-250)."""
    m, n, k = 16, 16, 140_000
    a = np.full((k, m), 127, np.int8)  # stored [k][lda=m]: A(m, k) = 127
    b = np.full((n, k), 127, np.int8)  # stored [n][ldb=k]
    c = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.INT32))
    spec = tpp.GemmSpec(m, n, k, m, k, m, in_dtype=tpp.DType.INT8, out_dtype=tpp.DType.INT32,
                        engine=tpp.Engine.TENSOR)
    tpp.brgemm(spec, tpp.BrgemmBatch.stride(to_dev(a.reshape(-1)), to_dev(b.reshape(-1)), 0, 0, 1), c)
    want = np.int64(127 * 127 * k)
    want32 = np.array([want & 0xFFFFFFFF], np.uint32).view(np.int32)[0]
    assert np.all(tpp.to_array(c) == want32) and want > 2**31
    k = 300
    a = np.full((k, 16), 127, np.int8)
    b = np.full((16, 304), 127, np.int8)
    c = tpp.alloc(tpp.TensorDesc(16, 16, 16, tpp.DType.INT32))
    spec = tpp.GemmSpec(16, 16, k, 16, 304, 16, in_dtype=tpp.DType.INT8, out_dtype=tpp.DType.INT32,
                        engine=tpp.Engine.TENSOR)
    tpp.brgemm(spec, tpp.BrgemmBatch.stride(to_dev(a.reshape(-1)), to_dev(b.reshape(-1)), 0, 0, 1), c)
    assert np.all(tpp.to_array(c) == 127 * 127 * 300)
    with pytest.raises(Exception):  # unaligned lda: the tensor engine refuses, AUTO would fall back
        spec = tpp.GemmSpec(15, 16, k, 15, 304, 15, in_dtype=tpp.DType.INT8, out_dtype=tpp.DType.INT32,
                            engine=tpp.Engine.TENSOR)
        tpp.brgemm(spec, tpp.BrgemmBatch.stride(to_dev(a.reshape(-1)), to_dev(b.reshape(-1)), 0, 0, 1),
                   tpp.alloc(tpp.TensorDesc(15, 16, 15, tpp.DType.INT32)))


def test_fc_gelu_epilogue_special_values():
    """The fused GELU epilogue on exact accumulators (identity weights: one
    non-zero product per output, so the tensor-core sum is exact) is bitwise
    the reference's GELU: range edges around |x| = 8, tiny, signed zero, large,
    +-inf and NaN (approx.py:267-276)."""
    rng = np.random.default_rng(33)
    Nb, bn, bc = 2, 64, 64
    specials = np.array([0.0, -0.0, 7.9921875, -7.9921875, 8.0, -8.0, 8.0625, -8.0625, 100.0, -100.0,
                         1e-30, -1e-30, 0.5, -0.5, 2.9, -2.9, 3.0e38, -3.0e38, np.inf, -np.inf, np.nan,
                         0.03125, -0.03125, 6.0, -6.0, 5.99, 1.0, -1.0], dtype=np.float32)
    x = rng.normal(0, 3, (Nb, 1, bn, bc)).astype(np.float32)
    flat = x.reshape(-1)
    flat[: specials.size] = specials
    xb = O.fp32_to_bf16_rne(x)
    eye = np.eye(64, dtype=np.float32)  # W[k, c]
    wv = np.zeros((1, 1, 32, 64, 2), dtype=np.uint16)
    wbits = O.fp32_to_bf16_rne(eye)
    for c in range(64):
        wv[0, 0, c // 2, :, c % 2] = wbits[:, c]
    layer = tpp.FcLayer(1, 1, 64, 64, to_dev(wv), activation=tpp.UnaryKind.GELU)
    out = layer.forward(to_dev(xb), Nb, bn)
    got = to_host(out).reshape(Nb, 1, bn, 64)
    want, _, _ = O.fc_forward_bf16(xb, wv, None, activation="gelu")
    assert bf16_equal(got.reshape(-1), np.asarray(want).reshape(-1))


def test_dilated_conv1d_atacworks_scale_bitwise():
    """The paper's ATACworks layer: W = 60400, Q = 60000,
    C = K = 15, S = 51, d = 8, FP32 — bitwise the reference order."""
    rng = np.random.default_rng(300)
    C_, K_, S_, d_, Q_ = 15, 15, 51, 8, 60000
    W_ = Q_ + (S_ - 1) * d_ + 0   # 60400
    x = rng.standard_normal((C_, W_)).astype(np.float32)
    wt = rng.standard_normal((C_ * S_, K_)).astype(np.float32)
    spec = tpp.DilatedConvSpec(C_, K_, W_, Q_, S_, d_)
    inp = tpp.TensorView(tpp.TensorDesc(C_, W_, C_, tpp.DType.FP32), to_dev(x.T.reshape(-1)))
    wv = tpp.TensorView(tpp.TensorDesc(C_ * S_, K_, C_ * S_, tpp.DType.FP32), to_dev(wt.T.reshape(-1)))
    out = tpp.alloc(tpp.TensorDesc(K_, Q_, K_, tpp.DType.FP32))
    tpp.dilated_conv1d_forward(spec, inp, wv, out)
    want = O.dilated_conv1d(x, wt, C_, K_, S_, d_, Q_)
    assert bits(tpp.to_array(out)) == bits(want)


@pytest.mark.parametrize("n", [4096 * 8, 1000])
def test_split_sgd_bf16_grads_bitwise(n):
    """split_sgd_step with BF16 gradients (kernels.py:235-251 accepts them;
    the data-parallel step exchanges BF16 dW buckets): the 16-byte vector
    kernel (n % 8 == 0) and the scalar one, bitwise the reference."""
    from paper_2104_05755_b200 import training as T
    rng = np.random.default_rng(400 + n)
    w = rng.standard_normal(n).astype(np.float32)
    g = O.fp32_to_bf16_rne((rng.standard_normal(n) * 1e-2).astype(np.float32))
    hi, lo = T.split_master(torch.from_numpy(w).cuda())
    tpp.split_sgd_flat(hi, lo, to_dev(g), 0.05)
    got = T.pack_master(hi, lo).cpu().numpy()
    want = O.split_sgd_step(w, O.bf16_to_fp32(g), 0.05)
    assert bits(got) == bits(np.asarray(want, np.float32))
