"""Pin the CPU oracle (oracle/tpp_oracle.py) to the reference's own outputs.

The fixtures were produced by the unmodified reference (tests/golden/make_golden.py);
every comparison here is bitwise unless stated.
"""

import numpy as np

from oracle import tpp_oracle as O


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8).tobytes()


def test_rne_matches_reference(golden):
    g = golden("dtypes.npz")
    got = O.fp32_to_bf16_rne(g["fp32_bits"].view(np.float32))
    assert np.array_equal(got, g["bf16_bits"])


def test_bf16_roundtrip_exhaustive():
    pats = np.arange(1 << 16, dtype=np.uint16)
    assert np.array_equal(O.fp32_to_bf16_rne(O.bf16_to_fp32(pats)), pats)


def test_cfg1_brgemm_bitwise(golden):
    g = golden("cfg1_brgemm.npz")
    m = n = k = 64
    a = [O.load_a(g["a"], i * m * k, m, k, m, "fp32") for i in range(16)]
    b = [O.load_b(g["b"], i * k * n, k, n, k, "fp32") for i in range(16)]
    c0 = g["c0"].reshape(n, m).T
    c = O.brgemm(a, b, c0, beta=1.0)
    assert bits(c.T.reshape(-1)) == bits(g["c"])


def _run_case(g, i):
    key = f"case{i:03d}"
    m, n, k, lda, ldb, ldc, cnt, sa, sb, vnni = (int(v) for v in g[key + "_meta"])
    dt = str(g[key + "_dtype"])
    beta = float(g[key + "_beta"])
    abuf, bbuf, c0 = g[key + "_a"], g[key + "_b"], g[key + "_c0"]
    a = [O.load_a(abuf, j * sa, m, k, lda, dt, vnni=bool(vnni)) for j in range(cnt)]
    b = [O.load_b(bbuf, j * sb, k, n, ldb, dt) for j in range(cnt)]
    c0w = c0.reshape(n, ldc).T[:m]
    c = O.brgemm(a, b, c0w, beta=beta, in_dtype=dt)
    full = c0.reshape(n, ldc).T.copy()
    full[:m] = c.astype(full.dtype)
    return full.T.reshape(-1), g[key + "_c"]


def test_brgemm_cases_bitwise(golden):
    g = golden("brgemm_cases.npz")
    for i in range(int(g["count"])):
        got, want = _run_case(g, i)
        assert bits(got) == bits(want), f"case {i}"


def test_gelu_table_fit_matches_reference(golden):
    g = golden("approx.npz")
    coeffs, base, range_max = O.GELU_TABLE
    assert np.array_equal(coeffs.view(np.uint32), g["gelu_coeffs"].view(np.uint32))
    assert base == int(g["gelu_base"]) and range_max == float(g["gelu_range_max"])


def test_gelu_and_grad_bitwise(golden):
    g = golden("approx.npz")
    assert bits(O.gelu(g["x"])) == bits(g["gelu"])
    assert bits(O.gelu_grad(g["x"])) == bits(g["gelu_grad"])


def test_exp_taylor_bitwise(golden):
    g = golden("approx.npz")
    got = O.exp_taylor(g["xe"])
    assert bits(got) == bits(g["exp"])


def test_eltwise_bitwise(golden):
    g = golden("eltwise.npz")
    x = g["x"]
    m, n = x.shape
    cm = lambda a: a.T.reshape(-1)  # column-major flat
    assert bits(cm(O.relu(x))) == bits(g["relu"])
    assert np.array_equal(O.bool_to_mask(O.relu_mask(x)), g["mask"])
    mb = O.mask_to_bool(g["mask"], m, n)
    assert bits(cm(O.relu_inv(g["dy"], mb))) == bits(g["relu_inv"])
    gel = O.fp32_to_bf16_rne(O.gelu(O.round_bf16(x)))
    assert np.array_equal(cm(gel), g["gelu_bf16"])
    assert bits(cm(g["dy"] * O.gelu_grad(x))) == bits(g["gelu_inv"])
    assert bits(cm(O.binary("add", x, g["bias"]))) == bits(g["add_bias"])
    assert bits(cm(O.muladd(x, g["y"], g["z"]))) == bits(g["muladd"])
    assert bits(cm(O.muladd(x, g["y"], g["z"], negate=True))) == bits(g["nmuladd"])
    assert bits(O.reduce_rows_sum(g["y"])) == bits(g["rsum"])
    assert bits(O.reduce_rows_sum(g["y"], squared=True)) == bits(g["rsumsq"])
    assert np.array_equal(O.vnni_pack(g["pats"], 2), g["vnni"])
    assert np.array_equal(O.vnni_to_vnnit(g["vnni"], 2, 2, 12, 10), g["vnnit"])
    assert np.array_equal(O.vnni_pack(g["pats_odd"], 2), g["vnni_odd"])
    assert np.array_equal(O.vnni_unpack(g["vnni_odd"], 2, 5, 7), g["pats_odd"])
    assert np.array_equal(cm(O.fp32_to_bf16_rne(x)), g["convert_bf16"])


def test_layernorm_matches_reference(golden):
    g = golden("layernorm.npz")
    for i in range(4):
        x = g[f"x{i}"]
        dt = str(g[f"dtype{i}"])
        xf = O.bf16_to_fp32(x) if dt == "bf16" else x
        out, mu, var = O.layernorm(xf, g[f"g{i}"], g[f"b{i}"], 1e-5)
        if dt == "bf16":
            out = O.fp32_to_bf16_rne(out)
        assert bits(out) == bits(g[f"out{i}"]), i
        assert bits(mu.astype(np.float32)) == bits(g[f"mean{i}"])
        assert bits(var.astype(np.float32)) == bits(g[f"var{i}"])


def test_softmax_and_split_sgd(golden):
    g = golden("softmax_sgd.npz")
    x = g["x"]
    want = g["y"]
    for j in range(6):
        sl = O.softmax_slice(x[:, j * 40:(j + 1) * 40])
        assert bits(sl.T.reshape(-1)) == bits(want[j * 40:(j + 1) * 40])
    x2 = g["x2"]
    want2 = g["y2"].reshape(99, 5).T
    for j in range(3):
        sl = O.softmax_slice(x2[:, j * 33:(j + 1) * 33])
        assert bits(sl) == bits(np.ascontiguousarray(want2[:, j * 33:(j + 1) * 33]))
    w = g["w0"]
    for gi in g["grads"]:
        w = O.split_sgd_step(w, gi, float(g["lr"]))
    assert bits(w) == bits(g["w1"])


def test_fc_fp32_and_bf16_compositions(golden):
    g = golden("fc.npz")
    for i in range(3):
        act = str(g[f"fp32_{i}_act"])
        c = O.fc_forward_fp32(g[f"fp32_{i}_a"], g[f"fp32_{i}_b"],
                              activation=None if act == "none" else act)
        assert bits(c) == bits(g[f"fp32_{i}_c"]), i
    for i in range(3):
        res = g[f"bf16_{i}_res"]
        out, _, _ = O.fc_forward_bf16(g[f"bf16_{i}_x"], g[f"bf16_{i}_w"], g[f"bf16_{i}_bias"],
                                      activation=str(g[f"bf16_{i}_act"]),
                                      residual_bits=res if res.size else None)
        assert np.array_equal(out, g[f"bf16_{i}_out"]), i


def test_conv_offset_composition(golden):
    g = golden("conv.npz")
    out, _ = O.conv2d_fwd_bf16(g["x"], g["w"])
    assert np.array_equal(out, g["out"])


def test_conv_strided_composition(golden):
    """Strided / 'valid' conv through the reference's own offset BRGEMM
    (fixture from tests/golden/make_golden.py gen_conv_strided), bitwise."""
    g = golden("conv_strided.npz")
    for name in ("s2_3x3", "s2_1x1", "s1_valid"):
        pad, st = (int(v) for v in g[f"{name}_geom"])
        out, _ = O.conv2d_fwd_bf16(g[f"{name}_x"], g[f"{name}_w"], pad=pad, stride=st)
        assert np.array_equal(out, g[f"{name}_out"]), name


def test_conv_bwd_data_adjoint(golden):
    """The FP64 backward-data restatement is the forward's adjoint:
    <conv(x), y> == <x, conv_bwd(y)> on the strided fixture shapes."""
    g = golden("conv_strided.npz")
    rng = np.random.default_rng(5)
    for name in ("s2_3x3", "s2_1x1", "s1_valid"):
        pad, st = (int(v) for v in g[f"{name}_geom"])
        x, w = g[f"{name}_x"], g[f"{name}_w"]
        _, acc = O.conv2d_fwd_bf16(x, w, pad=pad, stride=st)
        y = O.fp32_to_bf16_rne(rng.standard_normal(acc.shape).astype(np.float32))
        dx = O.conv2d_bwd_data_fp64(y, w, x.shape[2], x.shape[3], pad, st)
        lhs = float((acc.astype(np.float64) * O.bf16_to_fp32(y)).sum())
        rhs = float((O.bf16_to_fp32(x).astype(np.float64) * dx).sum())
        assert abs(lhs - rhs) <= 1e-5 * max(abs(lhs), 1e-30), (name, lhs, rhs)


def test_dilated_conv1d(golden):
    """The address-BRGEMM dilated conv of the reference, bitwise (kernels.py:350-378)."""
    g = golden("dilated.npz")
    for name in ("small", "atac"):
        c, k, s, d, w, q = (int(v) for v in g[f"{name}_shape"])
        out = O.dilated_conv1d(g[f"{name}_x"], g[f"{name}_w"], c, k, s, d, q)
        assert bits(out) == bits(g[f"{name}_out"]), name


def test_prng_and_dropout(golden):
    """PrngState seeding, uniform fills (incl. a 70001-row stream) and
    DROPOUT / DROPOUT_INV, bitwise (ops.py:195-236, 378-382, 430-444)."""
    g = golden("prng.npz")
    for s, want in zip(g["seeds"], g["seed_words"]):
        assert np.array_equal(O.prng_seed(int(s), 8), want)
    st = O.prng_seed(123, 6)
    assert bits(O.prng_uniform_block(st, 64).T.reshape(-1)) == bits(g["fill1"])
    f2 = O.prng_uniform_block(st, 37)
    assert bits(f2) == bits(O.strided2d(g["fill2"], 0, 37, 6, 40))
    assert np.array_equal(st, g["state_after"])
    lst = O.prng_seed(99, 3)
    lf = O.prng_uniform_block(lst, int(g["long_rows"]))
    assert bits(lf[g["long_idx"]]) == bits(g["long_sample"])
    assert np.array_equal(lst, g["long_state"])
    x = g["x"]
    m, n = x.shape
    dst = O.prng_seed(7, n)
    r1, k1 = O.dropout(x, dst, 0.3)
    r2, k2 = O.dropout(x, dst, 0.3)
    assert bits(r1.T.reshape(-1)) == bits(g["d1"]) and bits(r2.T.reshape(-1)) == bits(g["d2"])
    assert np.array_equal(O.bool_to_mask(k1), g["m1"]) and np.array_equal(O.bool_to_mask(k2), g["m2"])
    assert bits(O.dropout_inv(g["dy"], k1, 0.3).T.reshape(-1)) == bits(g["dinv"])
    assert bits(O.dropout_inv(g["dy"], k1, 1.0).T.reshape(-1)) == bits(g["dinv_p1"])
    xb = O.bf16_to_fp32(g["xb"]).reshape(n, m).T
    rb, kb = O.dropout(xb, O.prng_seed(5, n), 0.1)
    assert np.array_equal(O.fp32_to_bf16_rne(rb.T.reshape(-1)), g["db"])
    assert np.array_equal(O.bool_to_mask(kb), g["mb"])
    assert np.array_equal(O.prng_seed(5, 4), g["wrong_after"])  # wrong-width state untouched


def test_quantize_dequantize(golden):
    """ops.py:447-469 incl. ties-to-even, a NaN (scale 1, NaN -> 0), all-zero
    input and a caller scale that saturates."""
    g = golden("quant.npz")
    for name in ("uniform", "normal", "nan", "zeros", "ties"):
        x = g[name + "_x"]
        q, scale = O.quantize(x)
        assert scale == float(g[name + "_scale"]), name
        assert np.array_equal(q.T.reshape(-1), g[name + "_q"]), name
        assert bits(O.dequantize(q, scale).T.reshape(-1)) == bits(g[name + "_d"]), name
    q, _ = O.quantize(g["normal_x"], 0.01)
    assert np.array_equal(q.T.reshape(-1), g["given_q"])
