"""CPU-side tests: the C-ABI library loads and exports every header symbol,
host-side validation mirrors the reference's exceptions, and the product
path refuses to run without a GPU (no CPU fallback)."""

import ctypes
import os

import numpy as np
import pytest
import torch

import paper_2104_05755_b200 as tpp
from paper_2104_05755_b200 import _lib


def test_library_exports_every_header_symbol():
    lib = _lib.load(require_gpu=False)
    syms = _lib.header_symbols()
    assert len(syms) >= 24
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.tpp_version() == 1


def test_library_is_sm100a():
    # the .so embeds sm_100a SASS with tensor-core / TMA instructions
    data = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in data or b"compute_100a" in data


def test_c_abi_rejects_bad_specs_before_launch():
    lib = _lib.load(require_gpu=False)
    d = _lib.GemmDescC(2, 2, 2, 1, 2, 2, _lib.FP32, _lib.FP32, 0, 0, 0, 0, 0.0)  # lda < m
    assert lib.tpp_brgemm_stride(ctypes.byref(d), None, None, 0, 0, 1, None, None) == _lib.E_TENSOR
    assert b"lda" in lib.tpp_last_error()
    d = _lib.GemmDescC(2, 2, 2, 2, 2, 2, _lib.BF16, _lib.FP64, 0, 0, 0, 0, 0.0)
    assert lib.tpp_brgemm_stride(ctypes.byref(d), None, None, 0, 0, 1, None, None) == _lib.E_TENSOR
    d = _lib.GemmDescC(2, 2, 2, 2, 2, 2, _lib.FP32, _lib.FP32, 0, 1, 0, 0, 0.0)  # emulated fp32
    assert lib.tpp_brgemm_stride(ctypes.byref(d), None, None, 0, 0, 1, None, None) == _lib.E_TENSOR
    fc = _lib.FcDescC(1, 1, 1, 64, 64, 64, _lib.INT8, 0, 0, 0)
    assert lib.tpp_fc_forward(ctypes.byref(fc), None, None, None, None, None, None, None) == _lib.E_SPEC_DTYPE
    t = _lib.TensorDescC(4, 4, 4, _lib.FP32, 0)
    assert lib.tpp_unary(99, ctypes.byref(t), None, None, ctypes.byref(t), None, None, None) == _lib.E_SPEC_FLAG
    bad = _lib.TensorDescC(4, 4, 2, _lib.FP32, 0)  # ld < rows
    assert lib.tpp_binary(0, ctypes.byref(bad), None, ctypes.byref(t), None, ctypes.byref(t), None, None) == _lib.E_TENSOR
    assert lib.tpp_layernorm_blocked(1, 1, 1, 1, _lib.FP32, None, None, None, 1e-5, None, None, None, None) == _lib.E_TENSOR


def test_gemm_spec_validation_mirrors_reference():
    with pytest.raises(tpp.TensorError):
        tpp.GemmSpec(2, 2, 2, 1, 2, 2)  # lda < m
    with pytest.raises(tpp.TensorError):
        tpp.GemmSpec(2, 2, 2, 2, 2, 2, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP64)
    with pytest.raises(tpp.TensorError):
        tpp.GemmSpec(2, 2, 2, 2, 2, 2, compute_path=tpp.ComputePath.EMULATED_SPLIT)
    with pytest.raises(tpp.TensorError):
        tpp.GemmSpec(0, 2, 2, 2, 2, 2)
    s = tpp.GemmSpec(4, 4, 4, 4, 4, 4, in_dtype=tpp.DType.INT8, out_dtype=tpp.DType.INT32)
    assert s.alpha == 4 and s.acc_dtype is tpp.DType.INT32


def test_batch_constructors():
    a = torch.zeros(64)
    b = torch.zeros(64)
    st = tpp.BrgemmBatch.stride(a, b, 8, 4, 3)
    assert [o for _, o in st.a_refs] == [0, 8, 16] and [o for _, o in st.b_refs] == [0, 4, 8]
    of = tpp.BrgemmBatch.offset((a, 2), b, [0, 5], [1, 2])
    assert [o for _, o in of.a_refs] == [2, 7]
    with pytest.raises(tpp.TensorError):
        tpp.BrgemmBatch.address([a], [])
    with pytest.raises(tpp.TensorError):
        tpp.BrgemmBatch.offset(a, b, [0], [])


def test_tensor_desc_and_views():
    with pytest.raises(tpp.TensorError):
        tpp.TensorDesc(0, 1, 1, tpp.DType.FP32)
    with pytest.raises(tpp.TensorError):
        tpp.TensorDesc(4, 2, 3, tpp.DType.FP32)
    d = tpp.TensorDesc(3, 4, 5, tpp.DType.FP32)
    assert d.min_buffer_len == 5 * 3 + 3
    v = tpp.TensorView(d, torch.arange(18, dtype=torch.float32))
    assert v.as2d()[1, 2].item() == 1 + 2 * 5
    with pytest.raises(tpp.TensorError):
        tpp.TensorView(d, torch.zeros(10))
    with pytest.raises(tpp.TensorError):
        tpp.TensorView(d, torch.zeros(18, dtype=torch.float64))
    cb = v.col_block(1, 2)
    assert cb.as2d()[0, 0].item() == 5
    bc = tpp.broadcast(tpp.TensorView(tpp.TensorDesc(3, 1, 3, tpp.DType.FP32), torch.zeros(3)),
                       tpp.Bcast.COL, 3, 7)
    assert bc.desc.phys_cols == 1 and bc.logical2d().shape == (3, 7)
    with pytest.raises(tpp.TensorError):
        tpp.broadcast(v, tpp.Bcast.ROW, 3, 4)


def test_kernel_spec_inference_and_dispatch_cache():
    d = tpp.TensorDesc(8, 6, 8, tpp.DType.BF16)
    k = tpp.dispatch(tpp.KernelSpec(tpp.UnaryKind.RELU, (d,)))
    assert k.out_desc == tpp.TensorDesc(8, 6, 8, tpp.DType.BF16)
    assert tpp.dispatch(tpp.KernelSpec(tpp.UnaryKind.RELU, (d,))) is k
    r = tpp.infer_output_desc(tpp.KernelSpec(tpp.UnaryKind.REDUCE, (d,),
                                             reduce=tpp.ReduceSpec(tpp.ReduceAxis.ROWS, tpp.ReduceOp.SUM)))
    assert (r.rows, r.cols, r.dtype) == (8, 1, tpp.DType.FP32)
    v = tpp.infer_output_desc(tpp.KernelSpec(tpp.UnaryKind.TRANSFORM, (d,),
                                             transform=tpp.TransformSpec(tpp.TransformKind.VNNI, alpha=2)))
    assert (v.rows, v.cols) == (16, 3)
    with pytest.raises(tpp.InvalidSpecError) as e:
        tpp.infer_output_desc(tpp.KernelSpec(tpp.BinaryKind.ADD, (d, tpp.TensorDesc(3, 6, 3, tpp.DType.BF16))))
    assert e.value.code == "shape"
    with pytest.raises(tpp.InvalidSpecError):
        tpp.apply_ternary(tpp.TernaryKind.BRGEMM, None, None, None, None)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    """Compute on CPU-resident views must fail loudly, never silently run on the host."""
    d = tpp.TensorDesc(2, 2, 2, tpp.DType.FP32)
    a = tpp.TensorView(d, torch.ones(4))
    c = tpp.TensorView(d, torch.zeros(4))
    with pytest.raises(tpp.TppUnavailableError):
        tpp.gemm(tpp.GemmSpec(2, 2, 2, 2, 2, 2), a, tpp.TensorView(d, torch.ones(4)), c)
    with pytest.raises(tpp.TppUnavailableError):
        tpp.apply_unary(tpp.UnaryKind.RELU, a, c)
    assert torch.all(c.primary == 0)


def test_out_of_scope_kinds_refuse():
    d = tpp.TensorDesc(2, 2, 2, tpp.DType.FP32)
    a = tpp.TensorView(d, torch.ones(4))
    with pytest.raises(NotImplementedError):
        tpp.apply_unary(tpp.UnaryKind.TANH, a, a)
    with pytest.raises(NotImplementedError):
        tpp.apply_binary(tpp.BinaryKind.COMPARE, a, a, a)
