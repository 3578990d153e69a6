"""Known-answer GEMM/BRGEMM cases on the GPU, one per property the
reference's own GEMM tests pin (test_gemm.py: identity, the documented
order on FP64, beta = 0 / 1 / general, a one-entry BRGEMM with beta = 1,
VNNI vs plain A, the BF16 emulated-split path on a single product), each
checked bitwise."""

import numpy as np
import pytest
import torch

from oracle import tpp_oracle as O

pytestmark = pytest.mark.gpu

tpp = pytest.importorskip("paper_2104_05755_b200")


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield
    torch.cuda.synchronize()


def _spec(m, n, k, dtype=None, **kw):
    dtype = dtype or tpp.DType.FP32
    acc = {tpp.DType.FP64: tpp.DType.FP64, tpp.DType.INT8: tpp.DType.INT32}.get(dtype, tpp.DType.FP32)
    return tpp.GemmSpec(m, n, k, m, k, m, in_dtype=dtype, out_dtype=acc, **kw)


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8).tobytes()


def test_identity_times_x():
    x = np.arange(4, dtype=np.float32).reshape(2, 2)
    c = tpp.alloc(tpp.TensorDesc(2, 2, 2, tpp.DType.FP32))
    tpp.gemm(_spec(2, 2, 2), tpp.from_array(np.eye(2, dtype=np.float32)), tpp.from_array(x), c)
    assert _bits(tpp.to_array(c)) == _bits(x)


def test_fp64_follows_the_documented_order():
    """part = 0; part += a*b over ascending k (separately rounded); C = 0 + part."""
    rng = np.random.default_rng(11)
    m = n = k = 5
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((k, n))
    c = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.FP64))
    tpp.gemm(_spec(m, n, k, tpp.DType.FP64), tpp.from_array(a), tpp.from_array(b), c)
    want = np.zeros((m, n))
    for i in range(m):
        for j in range(n):
            part = 0.0
            for kk in range(k):
                part = part + a[i, kk] * b[kk, j]
            want[i, j] = 0.0 + part
    assert _bits(tpp.to_array(c)) == _bits(want)


def test_beta_one_adds_previous_contents():
    c = tpp.from_array(np.ones((2, 2), np.float32))
    tpp.gemm(_spec(2, 2, 2, beta=1.0), tpp.from_array(np.eye(2, dtype=np.float32)),
             tpp.from_array(np.full((2, 2), 3.0, np.float32)), c)
    assert tpp.to_array(c).tolist() == [[4.0, 4.0], [4.0, 4.0]]


def test_beta_zero_overwrites_nan():
    c = tpp.from_array(np.full((2, 2), np.nan, np.float32))
    tpp.gemm(_spec(2, 2, 2, beta=0.0), tpp.from_array(np.eye(2, dtype=np.float32)),
             tpp.from_array(np.ones((2, 2), np.float32)), c)
    assert tpp.to_array(c).tolist() == [[1.0, 1.0], [1.0, 1.0]]


def test_general_beta():
    c = tpp.from_array(np.full((2, 2), 2.0, np.float32))
    tpp.gemm(_spec(2, 2, 2, beta=0.5), tpp.from_array(np.eye(2, dtype=np.float32)),
             tpp.from_array(np.ones((2, 2), np.float32)), c)
    assert tpp.to_array(c).tolist() == [[2.0, 2.0], [2.0, 2.0]]


def test_one_entry_brgemm_with_beta_one_is_c_plus_gemm():
    rng = np.random.default_rng(12)
    m, n, k = 7, 5, 9
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    c0 = rng.standard_normal((m, n)).astype(np.float32)
    c = tpp.from_array(c0)
    av, bv = tpp.from_array(a), tpp.from_array(b)
    tpp.brgemm(_spec(m, n, k, beta=1.0), tpp.BrgemmBatch.stride(av.primary, bv.primary, 0, 0, 1), c)
    g = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.FP32))
    tpp.gemm(_spec(m, n, k), av, bv, g)
    # acc = C; part = A.B (from zero); acc + part, one rounding
    want = (c0 + tpp.to_array(g)).astype(np.float32)
    assert _bits(tpp.to_array(c)) == _bits(want)


@pytest.mark.parametrize("dtype,alpha", [("bf16", 2), ("int8", 4)])
def test_vnni_a_equals_plain_a(dtype, alpha):
    rng = np.random.default_rng(13)
    m, n, k = 6, 5, 10  # k not a multiple of alpha: zero-padded VNNI tail
    dt = tpp.DType.BF16 if dtype == "bf16" else tpp.DType.INT8
    if dtype == "bf16":
        a = rng.standard_normal((m, k)).astype(np.float32)
        b = rng.standard_normal((k, n)).astype(np.float32)
    else:
        a = rng.integers(-128, 128, (m, k), dtype=np.int8)
        b = rng.integers(-128, 128, (k, n), dtype=np.int8)
    av, bv = tpp.from_array(a, dt), tpp.from_array(b, dt)
    acc = tpp.DType.INT32 if dtype == "int8" else tpp.DType.FP32
    cp = tpp.alloc(tpp.TensorDesc(m, n, m, acc))
    tpp.gemm(_spec(m, n, k, dt, engine=tpp.Engine.ORDERED), av, bv, cp)
    packed = tpp.vnni_pack_a(av, alpha)
    cv = tpp.alloc(tpp.TensorDesc(m, n, m, acc))
    tpp.brgemm(_spec(m, n, k, dt, a_layout=tpp.ALayout.VNNI, engine=tpp.Engine.ORDERED),
               tpp.BrgemmBatch.stride(packed, bv.primary, 0, 0, 1), cv)
    assert _bits(tpp.to_array(cp)) == _bits(tpp.to_array(cv))


def test_bf16_single_product_native_and_emulated():
    a = tpp.from_array(np.array([[1.5]], np.float32), tpp.DType.BF16)
    b = tpp.from_array(np.array([[2.0]], np.float32), tpp.DType.BF16)
    for path in (tpp.ComputePath.NATIVE, tpp.ComputePath.EMULATED_SPLIT):
        c = tpp.alloc(tpp.TensorDesc(1, 1, 1, tpp.DType.FP32))
        tpp.gemm(_spec(1, 1, 1, tpp.DType.BF16, compute_path=path), a, b, c)
        assert float(tpp.to_array(c)[0, 0]) == 3.0


def test_bf16_emulated_matches_native_bitwise():
    """BF16 x BF16 products are exact in FP32, so the emulated split path
    (hi/lo halves) and the native path agree bit for bit (contraction.py)."""
    rng = np.random.default_rng(14)
    m = n = k = 8
    a = tpp.from_array(rng.standard_normal((m, k)).astype(np.float32), tpp.DType.BF16)
    b = tpp.from_array(rng.standard_normal((k, n)).astype(np.float32), tpp.DType.BF16)
    outs = []
    for path in (tpp.ComputePath.NATIVE, tpp.ComputePath.EMULATED_SPLIT):
        c = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.FP32))
        tpp.gemm(_spec(m, n, k, tpp.DType.BF16, compute_path=path, engine=tpp.Engine.ORDERED), a, b, c)
        outs.append(_bits(tpp.to_array(c)))
    assert outs[0] == outs[1]
    # and both equal the oracle's reference-order BRGEMM
    af = O.bf16_to_fp32(tpp.bits_of(a))
    bf = O.bf16_to_fp32(tpp.bits_of(b))
    want = O.brgemm([af], [bf], np.zeros((m, n), np.float32), beta=0.0)
    assert outs[0] == _bits(np.asarray(want, np.float32))
