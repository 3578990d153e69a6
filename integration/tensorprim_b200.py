"""Maintainer-side ctypes binding: what a `tensorprim` maintainer adds to call
the B200 BRGEMM path from inside the reference package.

It binds the C ABI of ``libtpp_b200.so`` (include/tpp_b200.h) directly — no
torch, no part of this repository's Python package — and translates a
``tensorprim.GemmSpec`` (contraction.py:44-85) into ``tpp_gemm_desc``.
Device pointers come from whatever array library the caller uses (torch,
cupy, ...).  Status codes map to the reference's exceptions
(tensor.py:29-30: TensorError for status 1; tpp_status in the header).
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_DEFAULT_LIB = os.path.join(_HERE, "..", "paper_2104_05755_b200", "libtpp_b200.so")


class GemmDesc(C.Structure):
    """include/tpp_b200.h: tpp_gemm_desc."""
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("k", C.c_int32), ("lda", C.c_int32),
                ("ldb", C.c_int32), ("ldc", C.c_int32), ("in_dtype", C.c_int32),
                ("out_dtype", C.c_int32), ("a_vnni", C.c_int32), ("compute_path", C.c_int32),
                ("engine", C.c_int32), ("reserved", C.c_int32), ("beta", C.c_double)]


# dtypes.py:17-24 DType values -> tpp_dtype codes (same order as the header)
DTYPE_CODE = {"fp64": 0, "fp32": 1, "bf16": 2, "int32": 3, "int16": 4, "int8": 5, "bit": 6}
ENGINE = {"auto": 0, "ordered": 1, "tensor": 2}


def load(path: str | None = None) -> C.CDLL:
    lib = C.CDLL(path or os.environ.get("TPP_B200_LIB", _DEFAULT_LIB))
    lib.tpp_last_error.restype = C.c_char_p
    lib.tpp_brgemm_stride.argtypes = [C.POINTER(GemmDesc), C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                      C.c_int64, C.c_void_p, C.c_void_p]
    lib.tpp_brgemm_stride.restype = C.c_int
    return lib


def desc_from_spec(spec, engine: str = "ordered") -> GemmDesc:
    """tensorprim.GemmSpec -> tpp_gemm_desc.  engine "ordered" keeps the
    reference's per-element order (bitwise); "auto" lets BF16 run on tcgen05."""
    return GemmDesc(spec.m, spec.n, spec.k, spec.lda, spec.ldb, spec.ldc,
                    DTYPE_CODE[spec.in_dtype.value], DTYPE_CODE[spec.out_dtype.value],
                    int(spec.a_layout.value == "vnni"), int(spec.compute_path.value == "emulated_split"),
                    ENGINE[engine], 0, float(spec.beta))


def _raise(lib, rc: int) -> None:
    msg = lib.tpp_last_error().decode(errors="replace")
    if rc == 1:
        try:
            from tensorprim import TensorError  # the reference's exception type
        except ImportError:
            TensorError = ValueError  # noqa: N806
        raise TensorError(msg)
    if rc == 7:
        raise NotImplementedError(msg)
    raise RuntimeError(f"tpp status {rc}: {msg}")


def brgemm_stride_device(lib, spec, a_dev_ptr: int, b_dev_ptr: int, stride_a: int, stride_b: int, count: int,
                         c_dev_ptr: int, stream: int = 0, engine: str = "ordered") -> None:
    """brgemm(spec, BrgemmBatch.stride(a, b, stride_a, stride_b, count), c)
    (contraction.py:162-168, 261-322) on device buffers."""
    d = desc_from_spec(spec, engine)
    rc = lib.tpp_brgemm_stride(C.byref(d), a_dev_ptr, b_dev_ptr, stride_a, stride_b, count, c_dev_ptr, stream)
    if rc:
        _raise(lib, rc)
