"""The BRGEMM TPP on the GPU — a drop-in for contraction.py of the reference
(/root/reference/pkg/src/tensorprim/contraction.py:1-347).

``brgemm(spec, batch, c)`` computes C = beta*C + sum_i A_i x B_i over the
three addressing variants of ``BrgemmBatch`` with the reference's argument
validation and exceptions.  The single-BRGEMM entry points run the ordered
SIMT kernel (K1), which reproduces the reference's per-element order and is
therefore bitwise identical for every dtype; blocking and thread count do
not change results, and they are accepted and ignored here as
the GPU owns the tiling.  Layer-level drivers (kernels.FcLayer, conv) run the
tcgen05 tensor-core BRGEMM.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
import enum
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .dtypes import DType
from .tensor import TensorDesc, TensorError, TensorView, may_share_memory


class ALayout(enum.Enum):
    PLAIN = "plain"
    VNNI = "vnni"


class ComputePath(enum.Enum):
    NATIVE = "native"
    EMULATED_SPLIT = "emulated_split"


class Engine(enum.Enum):
    """Which sm_100a engine runs a BRGEMM (not in the reference)."""
    AUTO = "auto"          # ordered SIMT for float BRGEMMs, tcgen05 kind::i8 for INT8 STRIDE
                           # batches (integer sums: any order is the reference's bits);
                           # tensor cores in the layer drivers
    ORDERED = "ordered"    # reference per-element order, bitwise parity
    TENSOR = "tensor"      # tcgen05 (layer drivers; INT8 STRIDE BRGEMMs)


@dataclass(frozen=True)
class GemmSpec:
    """contraction.py:44-85."""
    m: int
    n: int
    k: int
    lda: int
    ldb: int
    ldc: int
    in_dtype: DType = DType.FP32
    out_dtype: DType = DType.FP32
    beta: float = 0.0
    a_layout: ALayout = ALayout.PLAIN
    compute_path: ComputePath = ComputePath.NATIVE
    engine: Engine = Engine.AUTO

    def __post_init__(self):
        if min(self.m, self.n, self.k) < 1:
            raise TensorError("GEMM extents must be positive")
        if self.in_dtype not in (DType.FP64, DType.FP32, DType.BF16, DType.INT8):
            raise TensorError(f"unsupported input dtype {self.in_dtype}")
        if self.out_dtype is not self.acc_dtype:
            raise TensorError(f"output dtype must be {self.acc_dtype} for {self.in_dtype} inputs")
        if self.a_layout is ALayout.PLAIN and self.lda < self.m:
            raise TensorError("lda < M")
        if self.ldb < self.k:
            raise TensorError("ldb < K")
        if self.ldc < self.m:
            raise TensorError("ldc < M")
        if self.compute_path is ComputePath.EMULATED_SPLIT and self.in_dtype is not DType.BF16:
            raise TensorError("EMULATED_SPLIT applies to BF16 inputs")

    @property
    def acc_dtype(self) -> DType:
        if self.in_dtype is DType.FP64:
            return DType.FP64
        if self.in_dtype is DType.INT8:
            return DType.INT32
        return DType.FP32

    @property
    def alpha(self) -> int:
        return 4 if self.in_dtype is DType.INT8 else 2

    def c(self) -> _lib.GemmDescC:
        eng = {Engine.AUTO: _lib.ENGINE_AUTO, Engine.ORDERED: _lib.ENGINE_ORDERED,
               Engine.TENSOR: _lib.ENGINE_TENSOR}[self.engine]
        return _lib.GemmDescC(self.m, self.n, self.k, self.lda, self.ldb, self.ldc,
                              self.in_dtype.code, self.out_dtype.code,
                              int(self.a_layout is ALayout.VNNI),
                              int(self.compute_path is ComputePath.EMULATED_SPLIT), eng, 0,
                              float(self.beta))


@dataclass(frozen=True)
class BlockingParams:
    """contraction.py:88-96.  Results never depend on blocking; the GPU
    kernels choose their own tiles."""
    m_b: int
    n_b: int
    k_b: int

    def __post_init__(self):
        if min(self.m_b, self.n_b, self.k_b) < 1:
            raise TensorError("blocking factors must be positive")


DEFAULT_BLOCKING = {
    DType.FP64: BlockingParams(32, 6, 64),
    DType.FP32: BlockingParams(64, 6, 64),
    DType.BF16: BlockingParams(128, 6, 64),
    DType.INT8: BlockingParams(256, 6, 64),
}


class BatchKind(enum.Enum):
    ADDRESS = "address"
    OFFSET = "offset"
    STRIDE = "stride"


Ref = tuple  # (flat device buffer, element offset)


def _as_ref(x) -> Ref:
    """contraction.py:117-125."""
    if isinstance(x, TensorView):
        return (x.primary, 0)
    if isinstance(x, torch.Tensor):
        return (x, 0)
    buf, off = x
    if isinstance(buf, TensorView):
        buf = buf.primary
    return (buf, int(off))


class BrgemmBatch:
    """The (A_i, B_i) block sequence (contraction.py:128-168).  Device-side
    offset / pointer arrays are built once per batch and cached."""

    __slots__ = ("kind", "a_refs", "b_refs", "stride_a", "stride_b", "_dev")

    def __init__(self, kind: BatchKind, a_refs, b_refs, stride_a=0, stride_b=0):
        self.kind = kind
        self.a_refs = tuple(a_refs)
        self.b_refs = tuple(b_refs)
        self.stride_a = stride_a
        self.stride_b = stride_b
        self._dev = None

    @property
    def n(self) -> int:
        return len(self.a_refs)

    @staticmethod
    def address(a_refs: Sequence, b_refs: Sequence) -> "BrgemmBatch":
        a = tuple(_as_ref(r) for r in a_refs)
        b = tuple(_as_ref(r) for r in b_refs)
        if len(a) != len(b):
            raise TensorError(f"batch length mismatch: {len(a)} A blocks, {len(b)} B blocks")
        return BrgemmBatch(BatchKind.ADDRESS, a, b)

    @staticmethod
    def offset(a_base, b_base, a_offsets: Sequence[int], b_offsets: Sequence[int]) -> "BrgemmBatch":
        if len(a_offsets) != len(b_offsets):
            raise TensorError("offset batch length mismatch")
        ab, ao = _as_ref(a_base)
        bb, bo = _as_ref(b_base)
        return BrgemmBatch(BatchKind.OFFSET, tuple((ab, ao + int(o)) for o in a_offsets),
                           tuple((bb, bo + int(o)) for o in b_offsets))

    @staticmethod
    def stride(a_base, b_base, stride_a: int, stride_b: int, count: int) -> "BrgemmBatch":
        ab, ao = _as_ref(a_base)
        bb, bo = _as_ref(b_base)
        return BrgemmBatch(BatchKind.STRIDE,
                           tuple((ab, ao + i * int(stride_a)) for i in range(count)),
                           tuple((bb, bo + i * int(stride_b)) for i in range(count)),
                           int(stride_a), int(stride_b))

    def device_arrays(self, device, stream=None):
        """int64 arrays on the device: element offsets (OFFSET) or absolute
        addresses (ADDRESS).  Built once per batch: a pinned host staging
        buffer and an asynchronous copy on the issuing stream (no host
        synchronisation); later uses on other streams wait for that copy."""
        if self._dev is None:
            if self.kind is BatchKind.OFFSET:
                a = [o for _, o in self.a_refs]
                b = [o for _, o in self.b_refs]
            else:
                a = [buf.data_ptr() + o * buf.element_size() for buf, o in self.a_refs]
                b = [buf.data_ptr() + o * buf.element_size() for buf, o in self.b_refs]
            host = torch.tensor([a, b], dtype=torch.int64).pin_memory()
            s = stream if stream is not None else torch.cuda.current_stream(device)
            with torch.cuda.stream(s):
                dev = torch.empty((2, len(a)), dtype=torch.int64, device=device)
                dev.copy_(host, non_blocking=True)
            ev = None
            if not torch.cuda.is_current_stream_capturing():
                ev = torch.cuda.Event()
                ev.record(s)
            self._dev = (dev[0], dev[1], host, ev)
        a, b, _, ev = self._dev
        if ev is not None and not torch.cuda.is_current_stream_capturing():
            s = stream if stream is not None else torch.cuda.current_stream(device)
            s.wait_event(ev)
        return a, b


def _check_block(buf: torch.Tensor, off: int, rows: int, cols: int, ld: int, dtype: DType):
    """contraction.py:175-181 bounds rule."""
    if buf.dtype != dtype.storage:
        raise TensorError(f"block buffer dtype {buf.dtype} does not match {dtype}")
    need = off + ld * (cols - 1) + rows
    if off < 0 or need > buf.numel():
        raise TensorError(f"block exceeds buffer: need {need}, have {buf.numel()}")


def _check_vnni_block(buf: torch.Tensor, off: int, m: int, k: int, alpha: int, dtype: DType):
    """contraction.py:200-204."""
    if buf.dtype != dtype.storage:
        raise TensorError(f"block buffer dtype {buf.dtype} does not match {dtype}")
    groups = -(-k // alpha)
    if off < 0 or buf.numel() - off < groups * m * alpha:
        raise TensorError("VNNI block exceeds buffer")


def brgemm(spec: GemmSpec, batch: BrgemmBatch, c: TensorView,
           blocking: BlockingParams | None = None, threads: int = 1, stream=None) -> None:
    """C = beta*C + sum_i A_i x B_i (contraction.py:261-322), on the GPU.

    Validation (shape, dtype, ld, aliasing, block bounds) happens before any
    launch and raises the reference's TensorError.  ``blocking``/``threads``
    are accepted for API compatibility; results never depend on them.
    """
    if (c.desc.rows, c.desc.cols) != (spec.m, spec.n):
        raise TensorError(f"C must be {spec.m}x{spec.n}")
    if c.desc.dtype is not spec.out_dtype:
        raise TensorError(f"C dtype {c.desc.dtype} != {spec.out_dtype}")
    if c.desc.ld != spec.ldc:
        raise TensorError("C ld mismatch")
    for buf, _ in (*batch.a_refs, *batch.b_refs):
        if may_share_memory(c.primary, buf):
            raise TensorError("C must not alias any batch input")
    if blocking is not None and not isinstance(blocking, BlockingParams):
        raise TensorError("blocking must be BlockingParams")
    for buf, off in batch.a_refs:
        if spec.a_layout is ALayout.VNNI:
            _check_vnni_block(buf, off, spec.m, spec.k, spec.alpha, spec.in_dtype)
        else:
            _check_block(buf, off, spec.m, spec.k, spec.lda, spec.in_dtype)
    for buf, off in batch.b_refs:
        _check_block(buf, off, spec.k, spec.n, spec.ldb, spec.in_dtype)
    c.require_cuda("brgemm")
    for buf, _ in (*batch.a_refs, *batch.b_refs):
        if not buf.is_cuda:
            raise _lib.TppUnavailableError("brgemm: operands must live in CUDA memory")
    lib = _lib.load()
    d = spec.c()
    s = _lib.stream_ptr(stream)
    n = batch.n
    if n == 0 or batch.kind is BatchKind.STRIDE:
        if n == 0:
            a_ptr = b_ptr = 0
            sa = sb = 0
        else:
            (abuf, ao), (bbuf, bo) = batch.a_refs[0], batch.b_refs[0]
            a_ptr = abuf.data_ptr() + ao * abuf.element_size()
            b_ptr = bbuf.data_ptr() + bo * bbuf.element_size()
            sa, sb = batch.stride_a, batch.stride_b
        rc = lib.tpp_brgemm_stride(C.byref(d), a_ptr, b_ptr, sa, sb, n, c.ptr, s)
    elif batch.kind is BatchKind.OFFSET:
        ao, bo = batch.device_arrays(c.primary.device, stream)
        rc = lib.tpp_brgemm_offset(C.byref(d), batch.a_refs[0][0].data_ptr(),
                                   batch.b_refs[0][0].data_ptr(), ao.data_ptr(), bo.data_ptr(),
                                   n, c.ptr, s)
    else:
        ap, bp = batch.device_arrays(c.primary.device, stream)
        rc = lib.tpp_brgemm_address(C.byref(d), ap.data_ptr(), bp.data_ptr(), n, c.ptr, s)
    _lib.check(rc, "brgemm")


def gemm(spec: GemmSpec, a, b, c: TensorView, blocking: BlockingParams | None = None,
         threads: int = 1, stream=None) -> None:
    """contraction.py:325-329 — a one-entry batch."""
    brgemm(spec, BrgemmBatch.address([_as_ref(a)], [_as_ref(b)]), c, blocking, threads, stream)


def spec_for_views(a: TensorView, b: TensorView, c: TensorView, beta: float = 0.0,
                   a_layout: ALayout = ALayout.PLAIN,
                   compute_path: ComputePath = ComputePath.NATIVE) -> GemmSpec:
    """contraction.py:332-339."""
    return GemmSpec(m=a.desc.rows, n=b.desc.cols, k=a.desc.cols, lda=a.desc.ld, ldb=b.desc.ld,
                    ldc=c.desc.ld, in_dtype=a.desc.dtype, out_dtype=c.desc.dtype, beta=beta,
                    a_layout=a_layout, compute_path=compute_path)


def matmul(a: TensorView, b: TensorView, out: TensorView) -> None:
    """contraction.py:342-347 — GEMM with beta = 0."""
    if a.desc.cols != b.desc.rows:
        raise TensorError(f"matmul inner dims {a.desc.cols} != {b.desc.rows}")
    gemm(spec_for_views(a, b, out, beta=0.0), a, b, out)


def vnni_pack_a(a: TensorView, alpha: int) -> torch.Tensor:
    """contraction.py:238-247 on the GPU: a logical (M, K) view -> flat
    [ceil(K/alpha)][M][alpha] buffer (tail zero-padded), via the VNNI
    transform kernel."""
    from .ops import TransformKind, TransformSpec, transform
    from .tensor import alloc
    if alpha not in (2, 4):
        raise TensorError("alpha must be 2 (16-bit) or 4 (8-bit)")
    m, k = a.desc.rows, a.desc.cols
    groups = -(-k // alpha)
    out = alloc(TensorDesc(m * alpha, groups, m * alpha, a.desc.dtype), device=a.primary.device)
    transform(a, TransformSpec(TransformKind.VNNI, alpha=alpha), out)
    return out.primary


def vnni_unpack_a(flat: torch.Tensor, alpha: int, m: int, k: int) -> torch.Tensor:
    """contraction.py:250-254 — returns the logical (M, K) as a torch view."""
    groups = -(-k // alpha)
    grid = flat[:groups * m * alpha].reshape(groups, m, alpha)
    return grid.permute(1, 0, 2).reshape(m, groups * alpha)[:, :k]
