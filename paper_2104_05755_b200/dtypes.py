"""Element datatypes — the reference's ``DType`` (dtypes.py:17-73), with the
GPU storage each maps to.  BF16 is stored as ``torch.bfloat16`` (the same 16
bits the reference keeps as uint16 patterns, dtypes.py:1-8)."""

from __future__ import annotations

import enum

import numpy as np
import torch

from . import _lib


class DType(enum.Enum):
    FP64 = "fp64"
    FP32 = "fp32"
    BF16 = "bf16"
    INT32 = "int32"
    INT16 = "int16"
    INT8 = "int8"
    BIT = "bit"

    @property
    def bits(self) -> int:
        return _BITS[self]

    @property
    def storage(self) -> torch.dtype:
        """torch dtype of the device buffer."""
        return _TORCH[self]

    @property
    def np_storage(self) -> np.dtype:
        """numpy dtype the reference uses for the same buffer (dtypes.py:54-62)."""
        return _NP[self]

    @property
    def is_float(self) -> bool:
        return self in (DType.FP64, DType.FP32, DType.BF16)

    @property
    def code(self) -> int:
        """tpp_dtype value in the C ABI."""
        return _CODE[self]


_BITS = {DType.FP64: 64, DType.FP32: 32, DType.BF16: 16, DType.INT32: 32, DType.INT16: 16,
         DType.INT8: 8, DType.BIT: 1}
_TORCH = {DType.FP64: torch.float64, DType.FP32: torch.float32, DType.BF16: torch.bfloat16,
          DType.INT32: torch.int32, DType.INT16: torch.int16, DType.INT8: torch.int8,
          DType.BIT: torch.uint8}
_NP = {DType.FP64: np.dtype(np.float64), DType.FP32: np.dtype(np.float32),
       DType.BF16: np.dtype(np.uint16), DType.INT32: np.dtype(np.int32),
       DType.INT16: np.dtype(np.uint16), DType.INT8: np.dtype(np.int8),
       DType.BIT: np.dtype(np.uint8)}
_CODE = {DType.FP64: _lib.FP64, DType.FP32: _lib.FP32, DType.BF16: _lib.BF16,
         DType.INT32: _lib.INT32, DType.INT16: _lib.INT16, DType.INT8: _lib.INT8,
         DType.BIT: _lib.BIT}

# dtypes.py:64-73
COMPUTE_DTYPE = {DType.FP64: DType.FP64, DType.FP32: DType.FP32, DType.BF16: DType.FP32,
                 DType.INT32: DType.INT32, DType.INT16: DType.INT32, DType.INT8: DType.INT32}


def dtype_of_torch(t: torch.dtype) -> DType:
    for k, v in _TORCH.items():
        if v == t and k is not DType.BIT:
            return k
    if t == torch.uint8:
        return DType.BIT
    raise ValueError(f"no DType for {t}")
