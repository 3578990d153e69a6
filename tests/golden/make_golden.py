"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports ``tensorprim`` from /root/reference/pkg/src (read-only) through its
public API and writes ``tests/golden/*.npz``.  The fixtures pin the oracle
(``oracle/tpp_oracle.py``) and the GPU kernels to the reference's own outputs.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import tensorprim as tp  # noqa: E402
from tensorprim import approx  # noqa: E402
from tensorprim.dtypes import bf16_to_fp32, fp32_to_bf16_rne  # noqa: E402


def colmajor_flat(x):
    return np.asarray(x, order="F").reshape(-1, order="F").copy()


def save(name, **arrays):
    np.savez_compressed(os.path.join(OUT, name), **arrays)
    print("wrote", name, sum(a.nbytes for a in arrays.values()), "bytes raw")


def gen_dtypes():
    rng = np.random.default_rng(100)
    pats = rng.integers(0, 1 << 32, size=50_000, dtype=np.uint32)
    special = np.array([0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000,
                        0x7F800001, 0xFFC00000, 0x7F80FFFF, 0x7F7FFFFF, 0x3F808000,
                        0x3F818000, 0x3F800001, 0x00000001, 0x807FFFFF, 0x7FFF0000,
                        0x7F7F8000], dtype=np.uint32)
    pats = np.concatenate([special, pats])
    out = fp32_to_bf16_rne(pats.view(np.float32))
    save("dtypes.npz", fp32_bits=pats, bf16_bits=out.astype(np.uint16))


def gen_cfg1():
    """BASELINE cfg 1: 16 x (64x64) FP32 stride BRGEMM, beta=1, U[-1,1], seed 0."""
    rng = np.random.default_rng(0)
    m = n = k = 64
    cnt = 16
    a = rng.uniform(-1, 1, size=m * k * cnt).astype(np.float32)
    b = rng.uniform(-1, 1, size=k * n * cnt).astype(np.float32)
    c0 = rng.uniform(-1, 1, size=m * n).astype(np.float32)
    spec = tp.GemmSpec(m, n, k, m, k, m, beta=1.0)
    batch = tp.BrgemmBatch.stride(a, b, m * k, k * n, cnt)
    c = tp.TensorView(tp.TensorDesc(m, n, m, tp.DType.FP32), c0.copy())
    tp.brgemm(spec, batch, c)
    save("cfg1_brgemm.npz", a=a, b=b, c0=c0, c=np.array(c.primary))


def gen_brgemm_cases():
    """Random variant cases (verify.py:378-417 style) across dtypes / beta /
    VNNI / ld padding, recorded with the reference's own brgemm."""
    rng = np.random.default_rng(7)
    arrays = {}
    idx = 0
    for dtype, acc in ((tp.DType.FP32, tp.DType.FP32), (tp.DType.BF16, tp.DType.FP32),
                       (tp.DType.FP64, tp.DType.FP64), (tp.DType.INT8, tp.DType.INT32)):
        for case in range(12):
            m, n, k = (int(rng.integers(1, 40)) for _ in range(3))
            cnt = int(rng.integers(0, 7)) if case else 0
            beta = [0.0, 1.0, 0.5, -2.0][case % 4]
            vnni = dtype in (tp.DType.BF16, tp.DType.INT8) and case % 2 == 1
            alpha = 4 if dtype is tp.DType.INT8 else 2
            pad_a, pad_b, pad_c = (int(rng.integers(0, 3)) for _ in range(3))
            lda, ldb, ldc = m + pad_a, k + pad_b, m + pad_c
            if dtype is tp.DType.INT8:
                a_log = rng.integers(-128, 128, size=(cnt, m, k), dtype=np.int8)
                b_log = rng.integers(-128, 128, size=(cnt, k, n), dtype=np.int8)
                c0 = rng.integers(-1000, 1000, size=ldc * n).astype(np.int32)
                if beta not in (0.0, 1.0):
                    beta = 1.0
            elif dtype is tp.DType.BF16:
                a_log = fp32_to_bf16_rne(rng.standard_normal((cnt, m, k)).astype(np.float32))
                b_log = fp32_to_bf16_rne(rng.standard_normal((cnt, k, n)).astype(np.float32))
                c0 = rng.standard_normal(ldc * n).astype(np.float32)
            else:
                st = dtype.storage
                a_log = rng.standard_normal((cnt, m, k)).astype(st)
                b_log = rng.standard_normal((cnt, k, n)).astype(st)
                c0 = rng.standard_normal(ldc * n).astype(acc.storage)
            # flat buffers: A blocks (PLAIN col-major with lda, or VNNI), B blocks with ldb
            if vnni:
                ablocks = [tp.vnni_pack_a(a_log[i], alpha) for i in range(cnt)]
            else:
                ablocks = []
                for i in range(cnt):
                    blk = np.zeros((lda, k), dtype=a_log.dtype)
                    blk[:m] = a_log[i]
                    ablocks.append(colmajor_flat(blk))
            bblocks = []
            for i in range(cnt):
                blk = np.zeros((ldb, n), dtype=b_log.dtype)
                blk[:k] = b_log[i]
                bblocks.append(colmajor_flat(blk))
            sa = ablocks[0].size if cnt else 1
            sb = bblocks[0].size if cnt else 1
            abuf = np.concatenate(ablocks) if cnt else np.zeros(1, dtype=a_log.dtype)
            bbuf = np.concatenate(bblocks) if cnt else np.zeros(1, dtype=b_log.dtype)
            spec = tp.GemmSpec(m, n, k, lda if not vnni else m, ldb, ldc, in_dtype=dtype,
                               out_dtype=acc, beta=beta,
                               a_layout=tp.ALayout.VNNI if vnni else tp.ALayout.PLAIN)
            c = tp.TensorView(tp.TensorDesc(m, n, ldc, acc), c0.copy())
            tp.brgemm(spec, tp.BrgemmBatch.stride(abuf, bbuf, sa, sb, cnt), c)
            meta = np.array([m, n, k, lda if not vnni else m, ldb, ldc, cnt, sa, sb,
                             int(vnni)], dtype=np.int64)
            key = f"case{idx:03d}"
            arrays[key + "_meta"] = meta
            arrays[key + "_dtype"] = np.array(dtype.value)
            arrays[key + "_beta"] = np.array(beta, dtype=np.float64)
            arrays[key + "_a"] = abuf
            arrays[key + "_b"] = bbuf
            arrays[key + "_c0"] = c0
            arrays[key + "_c"] = np.array(c.primary)
            idx += 1
    arrays["count"] = np.array(idx)
    save("brgemm_cases.npz", **arrays)


def gen_approx():
    tabs = approx.coefficient_tables()
    gelu_tab = [t for t in tabs["minimax"] if t["name"] == "gelu_erf"][0]
    coeffs = np.array([[iv["coeffs"][j] for iv in gelu_tab["intervals"]] for j in range(4)],
                      dtype=np.float32)
    rng = np.random.default_rng(11)
    x = np.concatenate([
        np.linspace(-10, 10, 20001, dtype=np.float32),
        rng.standard_normal(20000).astype(np.float32) * 3,
        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 8.0, -8.0, 7.9999995, 1e-30,
                  -1e-30, 2 ** -5, 2 ** -6, 1.5 * 2 ** -5, 3.4e38, -3.4e38], dtype=np.float32),
    ])
    g = approx.gelu(x)
    gg = approx.gelu_grad(x)
    xe = np.concatenate([np.linspace(-100, 100, 40001, dtype=np.float32),
                         np.array([0.0, -0.0, 88.0, 88.5, -87.0, -87.5, np.inf, -np.inf],
                                  dtype=np.float32)])
    e = approx.exp_taylor(xe)
    save("approx.npz", gelu_coeffs=coeffs, gelu_base=np.array(gelu_tab["base"]),
         gelu_range_max=np.array(gelu_tab["range_max"]), x=x, gelu=g, gelu_grad=gg,
         xe=xe, exp=e)


def gen_eltwise():
    rng = np.random.default_rng(12)
    m, n = 37, 29
    x = rng.standard_normal((m, n)).astype(np.float32)
    x[0, :5] = [0.0, -0.0, np.nan, np.inf, -np.inf]
    xv = tp.from_array(x)
    out = tp.alloc(tp.TensorDesc(m, n, m, tp.DType.FP32))
    tp.apply_unary(tp.UnaryKind.RELU, xv, out, bitmask_output=True)
    relu_out = np.array(out.primary)
    mask = np.array(out.secondary)
    dy = rng.standard_normal((m, n)).astype(np.float32)
    dyv = tp.from_array(dy)
    dyv.secondary = mask
    dx = tp.alloc(tp.TensorDesc(m, n, m, tp.DType.FP32))
    tp.apply_unary(tp.UnaryKind.RELU_INV, dyv, dx)
    # bf16 in/out gelu through apply_unary (widen, compute, RNE narrow)
    xb = tp.from_array(x, tp.DType.BF16)
    gb = tp.alloc(tp.TensorDesc(m, n, m, tp.DType.BF16))
    tp.apply_unary(tp.UnaryKind.GELU, xb, gb)
    # gelu_inv: dy in primary, forward x in secondary
    dyg = tp.from_array(dy)
    dyg.secondary = np.array(tp.from_array(x).primary)
    gi = tp.alloc(tp.TensorDesc(m, n, m, tp.DType.FP32))
    tp.apply_unary(tp.UnaryKind.GELU_INV, dyg, gi)
    # bias add (COL broadcast) + muladd
    bias = rng.standard_normal((m, 1)).astype(np.float32)
    bb = tp.broadcast(tp.from_array(bias), tp.Bcast.COL, m, n)
    ad = tp.alloc(tp.TensorDesc(m, n, m, tp.DType.FP32))
    tp.apply_binary(tp.BinaryKind.ADD, xv, bb, ad)
    y = rng.standard_normal((m, n)).astype(np.float32)
    z = rng.standard_normal((m, n)).astype(np.float32)
    ma = tp.alloc(tp.TensorDesc(m, n, m, tp.DType.FP32))
    tp.apply_ternary(tp.TernaryKind.MULADD, xv, tp.from_array(y), tp.from_array(z), ma)
    nma = tp.alloc(tp.TensorDesc(m, n, m, tp.DType.FP32))
    tp.apply_ternary(tp.TernaryKind.NMULADD, xv, tp.from_array(y), tp.from_array(z), nma)
    # reduce rows sum / squared
    r1 = tp.alloc(tp.TensorDesc(m, 1, m, tp.DType.FP32))
    tp.reduce(tp.from_array(y), tp.ReduceSpec(tp.ReduceAxis.ROWS, tp.ReduceOp.SUM), r1)
    r2 = tp.alloc(tp.TensorDesc(m, 1, m, tp.DType.FP32))
    tp.reduce(tp.from_array(y), tp.ReduceSpec(tp.ReduceAxis.ROWS, tp.ReduceOp.SUM, True), r2)
    # transforms: VNNI, VNNI_TO_VNNIT, TRANSPOSE on bf16 patterns
    pats = rng.integers(0, 1 << 16, size=(12, 10), dtype=np.uint16)
    vn = tp.ops.vnni_pack(pats, 2)
    vnt = tp.ops.vnni_pack(tp.ops.vnni_unpack(vn, 2, 12, 10).T, 2)
    pats_odd = rng.integers(0, 1 << 16, size=(5, 7), dtype=np.uint16)
    vn_odd = tp.ops.vnni_pack(pats_odd, 2)
    # convert fp32 -> bf16 through the view API
    cv = tp.convert(tp.from_array(x), tp.DType.BF16)
    save("eltwise.npz", x=x, relu=relu_out, mask=mask, dy=dy, relu_inv=np.array(dx.primary),
         gelu_bf16=np.array(gb.primary), gelu_inv=np.array(gi.primary), bias=bias,
         add_bias=np.array(ad.primary), y=y, z=z, muladd=np.array(ma.primary),
         nmuladd=np.array(nma.primary), rsum=np.array(r1.primary), rsumsq=np.array(r2.primary),
         pats=pats, vnni=vn, vnnit=vnt, pats_odd=pats_odd, vnni_odd=vn_odd,
         convert_bf16=np.array(cv.primary))


def gen_layernorm():
    """kernels.layernorm on (features x tokens) views; the reference normalises
    each ROW of its 2-D view, so tokens are rows there."""
    rng = np.random.default_rng(13)
    arrays = {}
    for i, (m, n, dtype) in enumerate(((7, 48, tp.DType.FP32), (16, 1024, tp.DType.FP32),
                                       (32, 1024, tp.DType.BF16), (5, 64, tp.DType.BF16))):
        x = rng.standard_normal((m, n)).astype(np.float32) * (1 + i)
        x = x + np.float32(i * 0.5)
        xv = tp.from_array(x, dtype)
        gam = (1 + 0.1 * rng.standard_normal((1, n))).astype(np.float32)
        bet = (0.1 * rng.standard_normal((1, n))).astype(np.float32)
        if i == 2:
            gam[:] = 1.0
            bet[:] = 0.0
        g = tp.broadcast(tp.from_array(gam), tp.Bcast.ROW, m, n)
        b = tp.broadcast(tp.from_array(bet), tp.Bcast.ROW, m, n)
        out = tp.alloc(tp.TensorDesc(m, n, m, dtype))
        mo = tp.alloc(tp.TensorDesc(m, 1, m, tp.DType.FP32))
        vo = tp.alloc(tp.TensorDesc(m, 1, m, tp.DType.FP32))
        tp.layernorm(xv, g, b, 1e-5, out, mo, vo)
        arrays[f"x{i}"] = np.array(xv.primary).reshape(n, m).T.copy()
        arrays[f"g{i}"] = gam
        arrays[f"b{i}"] = bet
        arrays[f"out{i}"] = np.array(out.primary).reshape(n, m).T.copy()
        arrays[f"mean{i}"] = np.array(mo.primary)
        arrays[f"var{i}"] = np.array(vo.primary)
        arrays[f"dtype{i}"] = np.array(dtype.value)
    save("layernorm.npz", **arrays)


def gen_softmax_sgd():
    rng = np.random.default_rng(14)
    s1, s2, s3 = 1, 6, 40
    x = (rng.standard_normal((s1, s2 * s3)) * 4).astype(np.float32)
    y = tp.alloc(tp.TensorDesc(s1, s2 * s3, s1, tp.DType.FP32))
    tp.softmax(tp.SoftmaxSpec(s1, s2, s3), tp.from_array(x), y)
    x2 = rng.random((5, 3 * 33), dtype=np.float32)
    y2 = tp.alloc(tp.TensorDesc(5, 99, 5, tp.DType.FP32))
    tp.softmax(tp.SoftmaxSpec(5, 3, 33), tp.from_array(x2), y2)
    w0 = rng.standard_normal((8, 8)).astype(np.float32)
    split = tp.split_fp32(tp.from_array(w0))
    grads = rng.standard_normal((10, 8, 8)).astype(np.float32)
    for gi in grads:
        tp.kernels.split_sgd_step(split, tp.from_array(gi), 0.02)
    w1 = tp.to_array(tp.pack_fp32(split))
    save("softmax_sgd.npz", x=x, y=np.array(y.primary), x2=x2, y2=np.array(y2.primary),
         w0=w0, grads=grads, w1=w1, lr=np.array(0.02))


def gen_fc():
    rng = np.random.default_rng(15)
    arrays = {}
    # FP32 fc_forward with and without ReLU (kernels.py:300)
    for i, (mb, nb, kb, bm, bn, bk, act) in enumerate(((2, 3, 2, 4, 3, 5, "relu"),
                                                       (2, 2, 3, 8, 4, 8, None),
                                                       (1, 2, 4, 16, 8, 16, "relu"))):
        a4 = rng.standard_normal((mb, kb, bk, bm)).astype(np.float32)
        b4 = rng.standard_normal((nb, kb, bn, bk)).astype(np.float32)
        c = tp.alloc(tp.TensorDesc(bm, nb * mb * bn, bm, tp.DType.FP32))
        spec = tp.FcSpec(mb, nb, kb, bm, bn, bk,
                         activation=tp.UnaryKind.RELU if act else None)
        tp.fc_forward(spec, a4.reshape(-1), b4.reshape(-1), c)
        arrays[f"fp32_{i}_a"] = a4
        arrays[f"fp32_{i}_b"] = b4
        arrays[f"fp32_{i}_c"] = np.array(c.primary).reshape(nb, mb, bn, bm)
        arrays[f"fp32_{i}_act"] = np.array(act or "none")
    # BF16 FC composition per output block: brgemm(BF16, VNNI) -> +bias(COL)
    # -> act -> +residual -> convert(BF16)
    for i, (Nb, Cb, bn, bc, Kb, bk, act, res) in enumerate((
            (2, 3, 8, 16, 2, 16, "relu", False), (3, 2, 4, 8, 3, 8, "gelu", True),
            (2, 2, 32, 64, 2, 64, "relu", False))):
        x = fp32_to_bf16_rne(rng.normal(0, 1, size=(Nb, Cb, bn, bc)).astype(np.float32))
        wl = fp32_to_bf16_rne(rng.normal(0, 0.2, size=(Kb, Cb, bk, bc)).astype(np.float32))
        bias = fp32_to_bf16_rne(rng.normal(0, 0.2, size=(Kb * bk,)).astype(np.float32))
        resid = fp32_to_bf16_rne(rng.normal(0, 1, size=(Nb, Kb, bn, bk)).astype(np.float32))
        wv = np.stack([np.stack([tp.vnni_pack_a(wl[kb_, cb], 2) for cb in range(Cb)])
                       for kb_ in range(Kb)]).reshape(Kb, Cb, bc // 2, bk, 2)
        out = np.zeros((Nb, Kb, bn, bk), dtype=np.uint16)
        gspec = tp.GemmSpec(bk, bn, bc, bk, bc, bk, in_dtype=tp.DType.BF16,
                            out_dtype=tp.DType.FP32, beta=0.0, a_layout=tp.ALayout.VNNI)
        wflat = wv.reshape(-1)
        xflat = x.reshape(-1)
        for nb_ in range(Nb):
            for kb_ in range(Kb):
                cblk = tp.alloc(tp.TensorDesc(bk, bn, bk, tp.DType.FP32))
                batch = tp.BrgemmBatch.stride((wflat, kb_ * Cb * bc * bk),
                                              (xflat, nb_ * Cb * bn * bc),
                                              bc * bk, bn * bc, Cb)
                tp.brgemm(gspec, batch, cblk)
                bview = tp.TensorView(tp.TensorDesc(bk, 1, bk, tp.DType.BF16),
                                      bias[kb_ * bk:(kb_ + 1) * bk].copy())
                tp.apply_binary(tp.BinaryKind.ADD, cblk,
                                tp.broadcast(bview, tp.Bcast.COL, bk, bn), cblk)
                tp.apply_unary(tp.UnaryKind.RELU if act == "relu" else tp.UnaryKind.GELU,
                               cblk, cblk)
                if res:
                    rview = tp.TensorView(tp.TensorDesc(bk, bn, bk, tp.DType.BF16),
                                          resid[nb_, kb_].reshape(-1).copy())
                    tp.apply_binary(tp.BinaryKind.ADD, cblk, rview, cblk)
                ob = tp.convert(cblk, tp.DType.BF16)
                out[nb_, kb_] = np.array(ob.primary).reshape(bn, bk)
        arrays[f"bf16_{i}_x"] = x
        arrays[f"bf16_{i}_w"] = wv
        arrays[f"bf16_{i}_bias"] = bias
        arrays[f"bf16_{i}_res"] = resid if res else np.zeros(0, np.uint16)
        arrays[f"bf16_{i}_act"] = np.array(act)
        arrays[f"bf16_{i}_out"] = out
    save("fc.npz", **arrays)


def gen_conv():
    """3x3 'same' conv as OFFSET BRGEMM over (r, s, cb) taps on a padded input
    (contraction.py:152-160) — tiny shape; BF16 in, FP32 acc, BF16 out."""
    rng = np.random.default_rng(16)
    N, Cb, H, W, bc, Kb, bk, R, S = 2, 2, 5, 6, 8, 2, 8, 3, 3
    x = fp32_to_bf16_rne(rng.random((N, Cb, H, W, bc)).astype(np.float32))
    wl = fp32_to_bf16_rne(rng.normal(0, 0.3, size=(Kb, Cb, R, S, bk, bc)).astype(np.float32))
    wv = np.zeros((Kb, Cb, R, S, bc // 2, bk, 2), dtype=np.uint16)
    for kb_ in range(Kb):
        for cb in range(Cb):
            for r in range(R):
                for s in range(S):
                    wv[kb_, cb, r, s] = tp.vnni_pack_a(wl[kb_, cb, r, s], 2).reshape(bc // 2, bk, 2)
    Hp, Wp = H + 2, W + 2
    xp = np.zeros((N, Cb, Hp, Wp, bc), dtype=np.uint16)
    xp[:, :, 1:-1, 1:-1] = x
    xflat, wflat = xp.reshape(-1), wv.reshape(-1)
    out = np.zeros((N, Kb, H, W, bk), dtype=np.uint16)
    gspec = tp.GemmSpec(bk, W, bc, bk, bc, bk, in_dtype=tp.DType.BF16,
                        out_dtype=tp.DType.FP32, beta=0.0, a_layout=tp.ALayout.VNNI)
    for n in range(N):
        for kb_ in range(Kb):
            for oh in range(H):
                a_offs, b_offs = [], []
                for r in range(R):
                    for s in range(S):
                        for cb in range(Cb):
                            a_offs.append((((kb_ * Cb + cb) * R + r) * S + s) * bc * bk)
                            b_offs.append((((n * Cb + cb) * Hp + oh + r) * Wp + s) * bc)
                cblk = tp.alloc(tp.TensorDesc(bk, W, bk, tp.DType.FP32))
                tp.brgemm(gspec, tp.BrgemmBatch.offset(wflat, xflat, a_offs, b_offs), cblk)
                ob = tp.convert(cblk, tp.DType.BF16)
                out[n, kb_, oh] = np.array(ob.primary).reshape(W, bk)
    save("conv.npz", x=x, w=wv, out=out)


def gen_conv_strided():
    """Strided / non-'same' conv through the same composition: OFFSET BRGEMM
    over (r, s, cb) taps on an explicitly padded input, the tap's B block
    every stride-th padded column (ldb = stride * bc) of padded row
    oh * stride + r.  BF16 in, FP32 acc, BF16 out."""
    rng = np.random.default_rng(17)
    cases = {}
    for name, (N, Cb, H, W, bc, Kb, bk, R, S, pad, st) in {
            "s2_3x3": (2, 2, 7, 9, 8, 2, 8, 3, 3, 1, 2),
            "s2_1x1": (1, 2, 6, 6, 8, 1, 8, 1, 1, 0, 2),
            "s1_valid": (1, 1, 5, 6, 8, 2, 8, 3, 3, 0, 1)}.items():
        x = fp32_to_bf16_rne(rng.random((N, Cb, H, W, bc)).astype(np.float32))
        wl = fp32_to_bf16_rne(rng.normal(0, 0.3, size=(Kb, Cb, R, S, bk, bc)).astype(np.float32))
        wv = np.zeros((Kb, Cb, R, S, bc // 2, bk, 2), dtype=np.uint16)
        for kb_ in range(Kb):
            for cb in range(Cb):
                for r in range(R):
                    for s in range(S):
                        wv[kb_, cb, r, s] = tp.vnni_pack_a(wl[kb_, cb, r, s], 2).reshape(bc // 2, bk, 2)
        Hp, Wp = H + 2 * pad, W + 2 * pad
        P, Q = (Hp - R) // st + 1, (Wp - S) // st + 1
        xp = np.zeros((N, Cb, Hp, Wp, bc), dtype=np.uint16)
        xp[:, :, pad:pad + H, pad:pad + W] = x
        xflat, wflat = xp.reshape(-1), wv.reshape(-1)
        out = np.zeros((N, Kb, P, Q, bk), dtype=np.uint16)
        gspec = tp.GemmSpec(bk, Q, bc, bk, st * bc, bk, in_dtype=tp.DType.BF16,
                            out_dtype=tp.DType.FP32, beta=0.0, a_layout=tp.ALayout.VNNI)
        for n in range(N):
            for kb_ in range(Kb):
                for oh in range(P):
                    a_offs, b_offs = [], []
                    for r in range(R):
                        for s in range(S):
                            for cb in range(Cb):
                                a_offs.append((((kb_ * Cb + cb) * R + r) * S + s) * bc * bk)
                                b_offs.append((((n * Cb + cb) * Hp + oh * st + r) * Wp + s) * bc)
                    cblk = tp.alloc(tp.TensorDesc(bk, Q, bk, tp.DType.FP32))
                    tp.brgemm(gspec, tp.BrgemmBatch.offset(wflat, xflat, a_offs, b_offs), cblk)
                    ob = tp.convert(cblk, tp.DType.BF16)
                    out[n, kb_, oh] = np.array(ob.primary).reshape(Q, bk)
        cases.update({f"{name}_x": x, f"{name}_w": wv, f"{name}_out": out,
                      f"{name}_geom": np.array([pad, st], dtype=np.int64)})
    save("conv_strided.npz", **cases)


def gen_dilated():
    """1-D dilated conv (kernels.py:336-378) through the reference's own
    address-based BRGEMM driver: the reference test's shape and a wider
    ATACworks-like slice (C = K = 15, S = 51, d = 8)."""
    out = {}
    for name, (c, k, s, d, w, q, seed) in {"small": (3, 2, 5, 2, 28, 20, 15),
                                            "atac": (15, 15, 51, 8, 800, 400, 16)}.items():
        rng = np.random.default_rng(seed)
        x = rng.standard_normal((c, w)).astype(np.float32)
        wt = rng.standard_normal((c * s, k)).astype(np.float32)
        o = tp.alloc(tp.TensorDesc(k, q, k, tp.DType.FP32))
        tp.dilated_conv1d_forward(tp.DilatedConvSpec(c, k, w, q, s, d), tp.from_array(x), tp.from_array(wt), o)
        out[f"{name}_x"] = x
        out[f"{name}_w"] = wt
        out[f"{name}_out"] = tp.to_array(o).astype(np.float32)
        out[f"{name}_shape"] = np.array([c, k, s, d, w, q], dtype=np.int64)
    save("dilated.npz", **out)


def gen_prng():
    """PrngState seeding, PRNG fills and DROPOUT / DROPOUT_INV through the
    reference's apply_unary (ops.py:195-236, 326-328, 378-382, 430-444)."""
    P = tp.ops.PrngState
    seeds = np.array([0, 1, 123, 2024, (1 << 64) - 1], dtype=np.uint64)
    seed_words = np.stack([np.stack([P(int(s), 8).x, P(int(s), 8).y, P(int(s), 8).z, P(int(s), 8).w])
                           for s in seeds])
    # two successive PRNG fills from one state (the second continues the streams)
    src = tp.alloc(tp.TensorDesc(1, 1, 1, tp.DType.FP32))
    st = P(123, 6)
    src.tertiary = {"prng": st}
    f1 = tp.alloc(tp.TensorDesc(64, 6, 64, tp.DType.FP32))
    tp.apply_unary(tp.UnaryKind.PRNG, src, f1)
    f2 = tp.alloc(tp.TensorDesc(37, 6, 40, tp.DType.FP32))
    tp.apply_unary(tp.UnaryKind.PRNG, src, f2)
    state_after = np.stack([st.x, st.y, st.z, st.w])
    # a long fill: jump-ahead across many 64-row segments; keep sampled rows
    lst = P(99, 3)
    lsrc = tp.alloc(tp.TensorDesc(1, 1, 1, tp.DType.FP32))
    lsrc.tertiary = {"prng": lst}
    long_rows = 70_001
    lf = tp.alloc(tp.TensorDesc(long_rows, 3, long_rows, tp.DType.FP32))
    tp.apply_unary(tp.UnaryKind.PRNG, lsrc, lf)
    long_idx = np.concatenate([np.arange(0, long_rows, 997), np.arange(long_rows - 70, long_rows)])
    long_sample = tp.to_array(lf)[long_idx]
    long_state = np.stack([lst.x, lst.y, lst.z, lst.w])
    # dropout fp32, twice from one state, then the backward of the first
    rng = np.random.default_rng(16)
    m, n = 37, 29
    x = rng.standard_normal((m, n)).astype(np.float32)
    x[0, :4] = [np.nan, np.inf, -0.0, 0.0]
    xv = tp.from_array(x)
    dst = P(7, n)
    xv.tertiary = {"prng": dst}
    d1 = tp.alloc(tp.TensorDesc(m, n, m, tp.DType.FP32))
    tp.apply_unary(tp.UnaryKind.DROPOUT, xv, d1, dropout_p=0.3)
    d2 = tp.alloc(tp.TensorDesc(m, n, m, tp.DType.FP32))
    tp.apply_unary(tp.UnaryKind.DROPOUT, xv, d2, dropout_p=0.3)
    dy = rng.standard_normal((m, n)).astype(np.float32)
    dyv = tp.from_array(dy)
    dyv.secondary = d1.secondary
    di = tp.alloc(tp.TensorDesc(m, n, m, tp.DType.FP32))
    tp.apply_unary(tp.UnaryKind.DROPOUT_INV, dyv, di, dropout_p=0.3)
    di1 = tp.alloc(tp.TensorDesc(m, n, m, tp.DType.FP32))
    tp.apply_unary(tp.UnaryKind.DROPOUT_INV, dyv, di1, dropout_p=1.0)
    # bf16 in / out, p = 0.1; state built for the wrong width (fresh streams)
    xb = tp.from_array(x, tp.DType.BF16)
    wrong = P(5, 4)
    xb.tertiary = {"prng": wrong}
    db = tp.alloc(tp.TensorDesc(m, n, m, tp.DType.BF16))
    tp.apply_unary(tp.UnaryKind.DROPOUT, xb, db, dropout_p=0.1)
    wrong_after = np.stack([wrong.x, wrong.y, wrong.z, wrong.w])
    save("prng.npz", seeds=seeds, seed_words=seed_words, fill1=np.array(f1.primary),
         fill2=np.array(f2.primary), state_after=state_after, long_rows=np.int64(long_rows),
         long_idx=long_idx, long_sample=long_sample, long_state=long_state, x=x, dy=dy,
         d1=np.array(d1.primary), m1=np.array(d1.secondary), d2=np.array(d2.primary),
         m2=np.array(d2.secondary), dinv=np.array(di.primary), dinv_p1=np.array(di1.primary),
         xb=np.array(xb.primary), db=np.array(db.primary), mb=np.array(db.secondary),
         wrong_after=wrong_after)


def gen_quant():
    """QUANTIZE / DEQUANTIZE through the reference's apply_unary (ops.py:447-469)."""
    rng = np.random.default_rng(17)
    cases = {
        "uniform": rng.uniform(-2, 2, (8, 8)).astype(np.float32),
        "normal": (rng.standard_normal((37, 29)) * 3).astype(np.float32),
        "nan": rng.standard_normal((9, 5)).astype(np.float32),
        "zeros": np.zeros((4, 3), dtype=np.float32),
    }
    cases["nan"][2, 3] = np.nan
    # exact ties: amax 127 -> scale 1.0, so k + 0.5 must round to even
    ties = np.arange(-16, 16, dtype=np.float32).reshape(8, 4) + np.float32(0.5)
    ties[0, 0] = 127.0
    cases["ties"] = ties
    out = {}
    for name, x in cases.items():
        xv = tp.from_array(x)
        q = tp.alloc(tp.TensorDesc(x.shape[0], x.shape[1], x.shape[0], tp.DType.INT8))
        tp.apply_unary(tp.UnaryKind.QUANTIZE, xv, q)
        d = tp.alloc(tp.TensorDesc(x.shape[0], x.shape[1], x.shape[0], tp.DType.FP32))
        tp.apply_unary(tp.UnaryKind.DEQUANTIZE, q, d)
        out[name + "_x"] = x
        out[name + "_q"] = np.array(q.primary)
        out[name + "_scale"] = np.float64(q.tertiary["scale"])
        out[name + "_d"] = np.array(d.primary)
    # caller-provided scale (saturates at +-127)
    x = cases["normal"]
    xv = tp.from_array(x)
    xv.tertiary = {"scale": 0.01}
    q = tp.alloc(tp.TensorDesc(37, 29, 37, tp.DType.INT8))
    tp.apply_unary(tp.UnaryKind.QUANTIZE, xv, q)
    out["given_q"] = np.array(q.primary)
    save("quant.npz", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:   # only the named generators, e.g. `make_golden.py gen_conv_strided`
        for fn in sys.argv[1:]:
            globals()[fn]()
        sys.exit(0)
    gen_dtypes()
    gen_cfg1()
    gen_brgemm_cases()
    gen_approx()
    gen_eltwise()
    gen_layernorm()
    gen_softmax_sgd()
    gen_fc()
    gen_conv()
    gen_conv_strided()
    gen_dilated()
    gen_prng()
    gen_quant()
