"""The BRGEMM TPP on the GPU — a drop-in for contraction.py of the reference
(/root/reference/pkg/src/tensorprim/contraction.py:1-347).

``brgemm(spec, batch, c)`` computes C = beta*C + sum_i A_i x B_i over the
three addressing variants of ``BrgemmBatch`` with the reference's argument
validation and exceptions.  Engines (``GemmSpec.engine``):

* AUTO (default): BF16 batches run the tcgen05 BRGEMM (K11,
  brgemm_grouped.cu) for all three addressing variants — FP32 accumulation in TMEM over the whole batch,
  normwise <= 2e-2 of the reference (north_star's BF16 tolerance); INT8
  STRIDE batches run tcgen05 kind::i8 (exact); everything else runs the
  ordered SIMT engine (K1).
* ORDERED: K1 for every dtype — the reference's per-element order, bitwise.
* TENSOR: tensor cores or NotImplementedError.

Blocking and thread count never change results; they are
accepted and ignored, the GPU owns the tiling.  ``brgemm_grouped`` runs many
C blocks of one GemmSpec in one tcgen05 launch (the GPU form of composing a
layer from brgemm calls, kernels.py:312-329).
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
    AUTO = "auto"          # tcgen05 for aligned BF16 batches (all variants) and INT8 STRIDE
                           # batches; the ordered SIMT engine otherwise
    ORDERED = "ordered"    # reference per-element order, bitwise parity
    TENSOR = "tensor"      # tcgen05 (BF16 any variant, INT8 STRIDE) or NotImplementedError


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


def _tensor_eligible(spec: GemmSpec, a_refs, b_refs) -> bool:
    """The tcgen05 BRGEMM (K11) takes any non-empty BF16 batch: 16-byte
    aligned blocks with m, k, ldb (lda) multiples of 8 are staged with
    16-byte copies, any other block element-wise."""
    return spec.in_dtype is DType.BF16 and len(a_refs) > 0


class GroupedBatch:
    """Many independent BRGEMM batches of one GemmSpec, each feeding its own C
    block (group), for ``brgemm_grouped``.  Device index arrays are built once
    (pinned staging, asynchronous copy) and reused by every call.

    * ``stride(a, b, stride_a, stride_b, count, a_group_offsets, b_group_offsets)``:
      group g, entry i reads A at a + a_group_offsets[g] + i*stride_a (B alike);
    * ``offset(a, b, a_offsets, b_offsets)``: [groups][count] element offsets;
    * ``address(a_refs, b_refs)``: [groups][count] (buffer, offset) refs;
    * ``from_batches(batches)``: the narrowest of the three that describes a
      list of BrgemmBatch objects of equal length.
    """

    def __init__(self, kind: BatchKind, a_refs, b_refs, count: int, stride_a=0, stride_b=0,
                 a_goff=None, b_goff=None):
        self.kind = kind
        self.a_refs, self.b_refs = a_refs, b_refs      # [groups][count] (buffer, offset)
        self.count = count
        self.groups = len(a_refs)
        self.stride_a, self.stride_b = stride_a, stride_b
        self.a_goff, self.b_goff = a_goff, b_goff
        self._dev = None
        self._checked = set()   # (spec, C buffer, C offsets) combinations already validated
        self._gang = {}         # (m, n, device) -> gang tiling (or None)

    @staticmethod
    def stride(a_base, b_base, stride_a: int, stride_b: int, count: int,
               a_group_offsets: Sequence[int], b_group_offsets: Sequence[int]) -> "GroupedBatch":
        if len(a_group_offsets) != len(b_group_offsets):
            raise TensorError("group count mismatch")
        ab, ao = _as_ref(a_base)
        bb, bo = _as_ref(b_base)
        a_refs = [tuple((ab, ao + int(ga) + i * int(stride_a)) for i in range(count)) for ga in a_group_offsets]
        b_refs = [tuple((bb, bo + int(gb) + i * int(stride_b)) for i in range(count)) for gb in b_group_offsets]
        return GroupedBatch(BatchKind.STRIDE, a_refs, b_refs, count, int(stride_a), int(stride_b),
                            [ao + int(x) for x in a_group_offsets], [bo + int(x) for x in b_group_offsets])

    @staticmethod
    def offset(a_base, b_base, a_offsets, b_offsets) -> "GroupedBatch":
        ab, ao = _as_ref(a_base)
        bb, bo = _as_ref(b_base)
        if len(a_offsets) != len(b_offsets) or any(len(x) != len(y) for x, y in zip(a_offsets, b_offsets)):
            raise TensorError("offset batch length mismatch")
        count = len(a_offsets[0]) if len(a_offsets) else 0
        if any(len(x) != count for x in a_offsets):
            raise TensorError("every group needs the same batch length")
        a_refs = [tuple((ab, ao + int(o)) for o in row) for row in a_offsets]
        b_refs = [tuple((bb, bo + int(o)) for o in row) for row in b_offsets]
        return GroupedBatch(BatchKind.OFFSET, a_refs, b_refs, count)

    @staticmethod
    def address(a_refs, b_refs) -> "GroupedBatch":
        a = [tuple(_as_ref(r) for r in row) for row in a_refs]
        b = [tuple(_as_ref(r) for r in row) for row in b_refs]
        if len(a) != len(b) or any(len(x) != len(y) for x, y in zip(a, b)):
            raise TensorError("batch length mismatch")
        count = len(a[0]) if a else 0
        if any(len(x) != count for x in a):
            raise TensorError("every group needs the same batch length")
        # every A block in one buffer and every B block in one buffer: the
        # same blocks as offsets from those bases (the kernel's TMA staging
        # needs a base to build its views on; raw pointers get cp.async)
        if count and all(r[0] is a[0][0][0] for row in a for r in row) and \
                all(r[0] is b[0][0][0] for row in b for r in row):
            return GroupedBatch(BatchKind.OFFSET, a, b, count)
        return GroupedBatch(BatchKind.ADDRESS, a, b, count)

    @staticmethod
    def from_batches(batches: Sequence[BrgemmBatch]) -> "GroupedBatch":
        if not batches:
            raise TensorError("no batches")
        n = batches[0].n
        if any(bt.n != n for bt in batches):
            raise TensorError("every group needs the same batch length")
        kinds = {bt.kind for bt in batches}
        a0, b0 = batches[0].a_refs[0][0] if n else None, batches[0].b_refs[0][0] if n else None
        same_bufs = n > 0 and all(r[0] is a0 for bt in batches for r in bt.a_refs) and \
            all(r[0] is b0 for bt in batches for r in bt.b_refs)
        if kinds == {BatchKind.STRIDE} and same_bufs and len({(bt.stride_a, bt.stride_b) for bt in batches}) == 1:
            return GroupedBatch(BatchKind.STRIDE, [bt.a_refs for bt in batches], [bt.b_refs for bt in batches], n,
                                batches[0].stride_a, batches[0].stride_b,
                                [bt.a_refs[0][1] for bt in batches], [bt.b_refs[0][1] for bt in batches])
        if same_bufs:
            return GroupedBatch(BatchKind.OFFSET, [bt.a_refs for bt in batches], [bt.b_refs for bt in batches], n)
        return GroupedBatch(BatchKind.ADDRESS, [bt.a_refs for bt in batches], [bt.b_refs for bt in batches], n)

    def device_arrays(self, device, stream=None):
        """(a_index, b_index) device int64 arrays for the C ABI (see
        tpp_brgemm_grouped), built once on the issuing stream."""
        if self._dev is None:
            if self.kind is BatchKind.STRIDE:
                rows = [list(self.a_goff), list(self.b_goff)]
            elif self.kind is BatchKind.OFFSET:
                rows = [[o for grp in self.a_refs for _, o in grp], [o for grp in self.b_refs for _, o in grp]]
            else:
                rows = [[buf.data_ptr() + o * buf.element_size() for grp in self.a_refs for buf, o in grp],
                        [buf.data_ptr() + o * buf.element_size() for grp in self.b_refs for buf, o in grp]]
            host = torch.tensor(rows, dtype=torch.int64).pin_memory()
            s = stream if stream is not None else torch.cuda.current_stream(device)
            with torch.cuda.stream(s):
                dev = torch.empty(host.shape, dtype=torch.int64, device=device)
                dev.copy_(host, non_blocking=True)
            ev = None
            if not torch.cuda.is_current_stream_capturing():
                ev = torch.cuda.Event()
                ev.record(s)
            self._dev = (dev[0], dev[1], host, ev)
        a, b, _, ev = self._dev
        if ev is not None and not torch.cuda.is_current_stream_capturing():
            (stream if stream is not None else torch.cuda.current_stream(device)).wait_event(ev)
        return a, b


def _gang_table(keys_a, keys_b, m: int, n: int, device, sms: int):
    """Gang tiling of a grouped BRGEMM whose groups form a full cross product
    of A lists x B lists (the FC / conv compositions): returns (device int32
    table, ngangs, gang_m, gang_n) or None.  Gang rows pair two A lists
    (M = 128 MMAs) when m <= 64; gang columns take 2 or 4 B lists (N = 128 /
    256) when n <= 64, as wide as still leaves one gang per SM."""
    ia, ib = {}, {}
    ga = [ia.setdefault(k, len(ia)) for k in keys_a]
    gb = [ib.setdefault(k, len(ib)) for k in keys_b]
    na, nb = len(ia), len(ib)
    if m > 64 or na * nb != len(ga):
        return None
    cell = {}
    for g, (x, y) in enumerate(zip(ga, gb)):
        if (x, y) in cell:
            return None
        cell[(x, y)] = g
    gm = 2 if na >= 2 else 1
    gn = 1
    if n <= 64:
        for cand in (4, 2):
            if -(-na // gm) * -(-nb // cand) >= sms:
                gn = cand
                break
    if gm == 1 and gn == 1:
        return None
    rows, cols, cells = [], [], []
    row_rep = {x: g for (x, _), g in cell.items()}
    col_rep = {y: g for (_, y), g in cell.items()}
    for x0 in range(0, na, gm):
        for y0 in range(0, nb, gn):
            rows += [row_rep.get(x0 + i, -1) for i in range(gm)]
            cols += [col_rep.get(y0 + j, -1) for j in range(gn)]
            cells += [cell.get((x0 + i, y0 + j), -1) for i in range(gm) for j in range(gn)]
    ngangs = len(rows) // gm
    table = torch.tensor(rows + cols + cells, dtype=torch.int32).pin_memory().to(device, non_blocking=True)
    return table, ngangs, gm, gn


class _COffsets:
    """Per-group C offsets on the device, cached per (tensor, offsets)."""
    _cache: dict = {}

    @classmethod
    def get(cls, offs: tuple, device, stream):
        key = (offs, str(device))
        hit = cls._cache.get(key)
        if hit is None:
            host = torch.tensor(offs, dtype=torch.int64).pin_memory()
            s = stream if stream is not None else torch.cuda.current_stream(device)
            with torch.cuda.stream(s):
                dev = torch.empty(len(offs), dtype=torch.int64, device=device)
                dev.copy_(host, non_blocking=True)
            hit = (dev, host)
            if len(cls._cache) > 64:
                cls._cache.clear()
            cls._cache[key] = hit
        return hit[0]


def _check_grouped(spec: GemmSpec, gbatch: GroupedBatch, cbuf: torch.Tensor, c_offsets) -> None:
    """brgemm()'s validation (contraction.py:271-290) for every group, before any launch."""
    if len(c_offsets) != gbatch.groups:
        raise TensorError(f"{gbatch.groups} groups but {len(c_offsets)} C offsets")
    if len(set(int(o) for o in c_offsets)) != len(c_offsets):
        raise TensorError("C blocks of a grouped BRGEMM must be distinct")
    if cbuf.dtype != spec.out_dtype.storage:
        raise TensorError(f"C dtype {cbuf.dtype} != {spec.out_dtype}")
    for off in c_offsets:
        _check_block(cbuf, int(off), spec.m, spec.n, spec.ldc, spec.out_dtype)
    bufs = {id(buf): buf for grp in (*gbatch.a_refs, *gbatch.b_refs) for buf, _ in grp}
    for buf in bufs.values():
        if may_share_memory(cbuf, buf):
            raise TensorError("C must not alias any batch input")
    for grp in gbatch.a_refs:
        for buf, off in grp:
            if spec.a_layout is ALayout.VNNI:
                _check_vnni_block(buf, off, spec.m, spec.k, spec.alpha, spec.in_dtype)
            else:
                _check_block(buf, off, spec.m, spec.k, spec.lda, spec.in_dtype)
    for grp in gbatch.b_refs:
        for buf, off in grp:
            _check_block(buf, off, spec.k, spec.n, spec.ldb, spec.in_dtype)


def brgemm_grouped(spec: GemmSpec, gbatch: GroupedBatch, c, c_offsets: Sequence[int], stream=None) -> None:
    """For every group g: C_g = beta*C_g + sum_i A_{g,i} B_{g,i}, where C_g is
    the m x n (ldc) FP32 block at element offset c_offsets[g] of ``c`` —
    exactly ``brgemm(spec, batch_g, C_g)`` for each g (contraction.py:261-322),
    in ONE tcgen05 launch for aligned BF16 batches.  Other dtypes / layouts
    (and Engine.ORDERED) run one ordered brgemm call per group.  C blocks
    must be disjoint and must not alias any input block."""
    cbuf = c.primary if isinstance(c, TensorView) else c
    key = (spec, cbuf.data_ptr(), cbuf.numel(), cbuf.dtype, tuple(int(o) for o in c_offsets))
    if key not in gbatch._checked:
        _check_grouped(spec, gbatch, cbuf, c_offsets)
        gbatch._checked.add(key)
    if not cbuf.is_cuda:
        raise _lib.TppUnavailableError("brgemm_grouped: C must live in CUDA memory")
    if gbatch.groups == 0:
        return
    ekey = ("tc", spec)
    if ekey not in gbatch._checked and ("no-tc", spec) not in gbatch._checked:
        flat_a = [r for grp in gbatch.a_refs for r in grp]
        flat_b = [r for grp in gbatch.b_refs for r in grp]
        gbatch._checked.add(ekey if _tensor_eligible(spec, flat_a, flat_b) else ("no-tc", spec))
    use_tc = spec.engine is not Engine.ORDERED and ekey in gbatch._checked
    if not use_tc:
        if spec.engine is Engine.TENSOR:
            raise NotImplementedError("grouped tensor-core BRGEMM: BF16, count >= 1, m, k, ldb (lda) multiples "
                                      "of 8, 16-byte aligned blocks")
        for g in range(gbatch.groups):
            cv = TensorView(TensorDesc(spec.m, spec.n, spec.ldc, spec.out_dtype), cbuf[int(c_offsets[g]):])
            bt = BrgemmBatch(gbatch.kind, gbatch.a_refs[g], gbatch.b_refs[g], gbatch.stride_a, gbatch.stride_b)
            brgemm(spec, bt, cv, stream=stream)
        return
    lib = _lib.load()
    d = spec.c()
    d.engine = _lib.ENGINE_TENSOR
    dev = cbuf.device
    ai, bi = gbatch.device_arrays(dev, stream)
    coff = _COffsets.get(tuple(int(o) for o in c_offsets), dev, stream)
    kind = {BatchKind.STRIDE: 0, BatchKind.OFFSET: 1, BatchKind.ADDRESS: 2}[gbatch.kind]
    if kind == 2:
        a_ptr = b_ptr = 0
    else:
        (abuf, _), (bbuf, _) = gbatch.a_refs[0][0], gbatch.b_refs[0][0]
        a_ptr, b_ptr = abuf.data_ptr(), bbuf.data_ptr()
    gkey = ("gang", spec.m, spec.n, str(dev))
    if gkey not in gbatch._gang:
        # groups sharing A lists (rows) and B lists (columns): tiled together
        if gbatch.kind is BatchKind.STRIDE:
            ka, kb = list(gbatch.a_goff), list(gbatch.b_goff)
        else:
            ka = [tuple((id(buf), o) for buf, o in grp) for grp in gbatch.a_refs]
            kb = [tuple((id(buf), o) for buf, o in grp) for grp in gbatch.b_refs]
        gbatch._gang[gkey] = _gang_table(ka, kb, spec.m, spec.n, dev, int(lib.tpp_device_sm_count()))
    gang = gbatch._gang[gkey]
    if gang is not None:
        table, ngangs, gm, gn = gang
        rc = lib.tpp_brgemm_grouped_gang(C.byref(d), kind, a_ptr, b_ptr, gbatch.stride_a, gbatch.stride_b,
                                         ai.data_ptr(), bi.data_ptr(), gbatch.count, cbuf.data_ptr(),
                                         coff.data_ptr(), gbatch.groups, table.data_ptr(), ngangs, gm, gn,
                                         _lib.stream_ptr(stream))
    else:
        rc = lib.tpp_brgemm_grouped(C.byref(d), kind, a_ptr, b_ptr, gbatch.stride_a, gbatch.stride_b,
                                    ai.data_ptr(), bi.data_ptr(), gbatch.count, cbuf.data_ptr(), coff.data_ptr(),
                                    gbatch.groups, _lib.stream_ptr(stream))
    _lib.check(rc, "brgemm_grouped")


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
