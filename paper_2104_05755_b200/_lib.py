"""ctypes binding of ``libtpp_b200.so`` (the C ABI in include/tpp_b200.h).

The product path has no fallback: if the library or a CUDA device is
missing, every compute call raises ``TppUnavailableError``.
"""

from __future__ import annotations

import ctypes as C
import os
import re
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtpp_b200.so")
HEADER = os.path.join(HERE, "..", "include", "tpp_b200.h")

# status codes (tpp_status)
OK, E_TENSOR, E_SPEC_SHAPE, E_SPEC_DTYPE, E_SPEC_FLAG, E_INDEX, E_CUDA, E_UNSUPPORTED = range(8)
# dtypes (tpp_dtype) — same order as dtypes.py:17-24
FP64, FP32, BF16, INT32, INT16, INT8, BIT = range(7)
BCAST_NONE, BCAST_ROW, BCAST_COL, BCAST_SCALAR = range(4)
ENGINE_AUTO, ENGINE_ORDERED, ENGINE_TENSOR = range(3)
ACT_NONE, ACT_RELU, ACT_GELU = range(3)
FC_BIAS, FC_RESIDUAL, FC_RELU_MASK, FC_OUT_FP32, FC_BIAS_FP32, FC_RELU_INV, FC_SGD = 1, 2, 4, 8, 16, 32, 64
FC_DYNAMIC_TILES = 128


class TppUnavailableError(RuntimeError):
    """The sm_100a library or a CUDA device is not available."""


class TensorDescC(C.Structure):
    _fields_ = [("rows", C.c_int32), ("cols", C.c_int32), ("ld", C.c_int32),
                ("dtype", C.c_int32), ("bcast", C.c_int32)]


class GemmDescC(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("k", C.c_int32), ("lda", C.c_int32),
                ("ldb", C.c_int32), ("ldc", C.c_int32), ("in_dtype", C.c_int32),
                ("out_dtype", C.c_int32), ("a_vnni", C.c_int32), ("compute_path", C.c_int32),
                ("engine", C.c_int32), ("reserved", C.c_int32), ("beta", C.c_double)]


class FcDescC(C.Structure):
    _fields_ = [("m_b", C.c_int32), ("n_b", C.c_int32), ("k_b", C.c_int32), ("bm", C.c_int32),
                ("bn", C.c_int32), ("bk", C.c_int32), ("in_dtype", C.c_int32),
                ("activation", C.c_int32), ("flags", C.c_int32), ("block_n", C.c_int32)]


class ConvDescC(C.Structure):
    _fields_ = [("n", C.c_int32), ("c_b", C.c_int32), ("k_b", C.c_int32), ("h", C.c_int32),
                ("w", C.c_int32), ("r", C.c_int32), ("s", C.c_int32), ("pad", C.c_int32),
                ("bc", C.c_int32), ("bk", C.c_int32), ("flags", C.c_int32),
                ("reserved", C.c_int32)]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_SIGS = {
    "tpp_last_error": (C.c_char_p, []),
    "tpp_last_config": (C.c_char_p, []),
    "tpp_version": (C.c_int, []),
    "tpp_device_sm_count": (C.c_int, []),
    "tpp_brgemm_stride": (C.c_int, [C.POINTER(GemmDescC), _P, _P, _I64, _I64, _I64, _P, _P]),
    "tpp_brgemm_offset": (C.c_int, [C.POINTER(GemmDescC), _P, _P, _P, _P, _I64, _P, _P]),
    "tpp_brgemm_address": (C.c_int, [C.POINTER(GemmDescC), _P, _P, _I64, _P, _P]),
    "tpp_brgemm_grouped": (C.c_int, [C.POINTER(GemmDescC), _I32, _P, _P, _I64, _I64, _P, _P, _I64, _P, _P,
                                     _I64, _P]),
    "tpp_brgemm_grouped_gang": (C.c_int, [C.POINTER(GemmDescC), _I32, _P, _P, _I64, _I64, _P, _P, _I64, _P, _P,
                                          _I64, _P, _I32, _I32, _I32, _P]),
    "tpp_brgemm_grouped_bf16": (C.c_int, [C.POINTER(GemmDescC), _I32, _P, _P, _I64, _I64, _P, _P, _I64, _P, _P,
                                          _I64, _P, _I32, _I32, _I32, _I32, _I32, _P]),
    "tpp_brgemm_stride_batched": (C.c_int, [C.POINTER(GemmDescC), _P, _P, _I64, _I64, _I64, _P,
                                            _I64, _I64, _I64, _I64, _P]),
    "tpp_fc_packed_weight_bytes": (C.c_int64, [C.POINTER(FcDescC)]),
    "tpp_fc_pack_weights": (C.c_int, [C.POINTER(FcDescC), _P, _P, _P]),
    "tpp_fc_forward": (C.c_int, [C.POINTER(FcDescC), _P, _P, _P, _P, _P, _P, _P]),
    "tpp_fc_backward_data": (C.c_int, [C.POINTER(FcDescC), _P, _P, _P, _P, _P]),
    "tpp_fc_backward_weights": (C.c_int, [C.POINTER(FcDescC), _P, _P, _P, _P]),
    "tpp_fc_backward_weights_sgd": (C.c_int, [C.POINTER(FcDescC), _P, _P, _P, _P, C.c_float, _P]),
    "tpp_softmax_xent_blocked": (C.c_int, [_I32, _I32, _I32, _I32, _P, _P, C.c_float, _P, _P, _P]),
    "tpp_conv_packed_weight_bytes": (C.c_int64, [C.POINTER(ConvDescC)]),
    "tpp_conv_pack_weights": (C.c_int, [C.POINTER(ConvDescC), _P, _P, _I32, _P]),
    "tpp_conv_forward": (C.c_int, [C.POINTER(ConvDescC), _P, _P, _P, _P]),
    "tpp_conv_pad": (C.c_int, [_I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P, _P, _P]),
    "tpp_conv_backward_data": (C.c_int, [C.POINTER(ConvDescC), _P, _P, _P, _P]),
    "tpp_conv_backward_weights_workspace_bytes": (C.c_int64, [C.POINTER(ConvDescC)]),
    "tpp_conv_backward_weights": (C.c_int, [C.POINTER(ConvDescC), _P, _P, _P, _P, _P]),
    "tpp_unary": (C.c_int, [_I32, C.POINTER(TensorDescC), _P, _P, C.POINTER(TensorDescC), _P,
                            _P, _P]),
    "tpp_binary": (C.c_int, [_I32, C.POINTER(TensorDescC), _P, C.POINTER(TensorDescC), _P,
                             C.POINTER(TensorDescC), _P, _P]),
    "tpp_ternary": (C.c_int, [_I32, C.POINTER(TensorDescC), _P, C.POINTER(TensorDescC), _P,
                              C.POINTER(TensorDescC), _P, C.POINTER(TensorDescC), _P, _P]),
    "tpp_reduce": (C.c_int, [C.POINTER(TensorDescC), _P, _I32, _I32, _I32,
                             C.POINTER(TensorDescC), _P, _P]),
    "tpp_transform": (C.c_int, [_I32, C.POINTER(TensorDescC), _P, _I32, _I32, _I32, _I32,
                                C.POINTER(TensorDescC), _P, _P]),
    "tpp_convert": (C.c_int, [C.POINTER(TensorDescC), _P, C.POINTER(TensorDescC), _P, _P]),
    "tpp_layernorm": (C.c_int, [C.POINTER(TensorDescC), _P, C.POINTER(TensorDescC), _P,
                                C.POINTER(TensorDescC), _P, C.c_double, C.POINTER(TensorDescC),
                                _P, _P, _P, _P]),
    "tpp_layernorm_blocked": (C.c_int, [_I32, _I32, _I32, _I32, _I32, _P, _P, _P, C.c_double, _P,
                                        _P, _P, _P]),
    "tpp_layernorm_blocked_ex": (C.c_int, [_I32, _I32, _I32, _I32, _I32, _P, _P, _P, C.c_double, _P,
                                        _P, _P, _I32, _P]),
    "tpp_softmax": (C.c_int, [_I32, _I32, _I32, C.POINTER(TensorDescC), _P,
                              C.POINTER(TensorDescC), _P, _P]),
    "tpp_split_sgd": (C.c_int, [_I64, _P, _P, _P, _I32, C.c_float, _P]),
    "tpp_debug_phase_timestamps": (C.c_int, [_P]),
    "tpp_set_tile_scheduling": (C.c_int, [C.c_int32]),
    "tpp_quantize": (C.c_int, [C.POINTER(TensorDescC), _P, _I32, C.c_double,
                               C.POINTER(TensorDescC), _P, _P, _P, _P]),
    "tpp_dequantize": (C.c_int, [C.POINTER(TensorDescC), _P, C.c_double,
                                 C.POINTER(TensorDescC), _P, _P]),
    "tpp_prng_seed": (C.c_int, [C.c_uint64, _I32, _P, _P]),
    "tpp_prng_fill": (C.c_int, [_P, _P, C.POINTER(TensorDescC), _P, _P]),
    "tpp_dropout": (C.c_int, [C.POINTER(TensorDescC), _P, _P, _P, C.c_double,
                              C.POINTER(TensorDescC), _P, _P, _P]),
    "tpp_dropout_inv": (C.c_int, [C.POINTER(TensorDescC), _P, _P, C.c_double,
                                  C.POINTER(TensorDescC), _P, _P]),
}

_lib = None
_lock = threading.Lock()


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tpp_[a-z0-9_]+)\s*\(", src)))


def load(require_gpu: bool = True):
    """Load the library (once).  With ``require_gpu`` also insist on a CUDA
    device — the compute entry points have no CPU fallback."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise TppUnavailableError(
                    f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_gpu:
        import torch
        if not torch.cuda.is_available():
            raise TppUnavailableError("no CUDA device: the TPP kernels run on sm_100a only")
    return _lib


def check(status: int, what: str = "") -> None:
    """Map a tpp_status to the reference's exception types."""
    if status == OK:
        return
    msg = _lib.tpp_last_error().decode(errors="replace") if _lib is not None else ""
    msg = f"{what}: {msg}" if what else msg
    from .tensor import TensorError
    from .ops import InvalidSpecError
    if status == E_TENSOR:
        raise TensorError(msg)
    if status == E_SPEC_SHAPE:
        raise InvalidSpecError("shape", msg)
    if status == E_SPEC_DTYPE:
        raise InvalidSpecError("dtype", msg)
    if status == E_SPEC_FLAG:
        raise InvalidSpecError("flag", msg)
    if status == E_INDEX:
        raise IndexError(msg)
    if status == E_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"CUDA error in TPP library: {msg}")


def last_config() -> str:
    """Instantiation / grid of the last tensor-core kernel launched by this
    thread (tpp_last_config), e.g. 'brgemm_tc_kernel<256,3,2,0,2,1> grid=148 ...'."""
    return load(require_gpu=False).tpp_last_config().decode()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
