"""Unary / binary / ternary TPPs, reduce, transforms and the dispatch cache on
the GPU — a drop-in for ops.py of the reference
(/root/reference/pkg/src/tensorprim/ops.py).

Same operator enums, argument order, output-shape inference and exceptions.
The kinds on the BRGEMM hot path
run as sm_100a kernels, bitwise identical to the reference; kinds outside
that scope (gather/scatter, tanh/sigmoid, shuffle transpose) raise
NotImplementedError instead of silently running elsewhere.  PRNG / DROPOUT /
DROPOUT_INV run on the GPU with the reference's per-column
xorshift128 streams, bitwise; QUANTIZE / DEQUANTIZE (the INT8 BRGEMM's
neighbours) likewise.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
import enum
import threading
from typing import Optional, Sequence

import torch

from . import _lib
from .dtypes import DType
from .tensor import (Bcast, TensorDesc, TensorError, TensorView, alloc_bitmask,
                     bitmask_bytes)


class UnaryKind(enum.Enum):
    IDENTITY = "identity"
    ZERO = "zero"
    SQUARE = "square"
    INC = "inc"
    DEC = "dec"
    SQRT = "sqrt"
    RECIPROCAL = "reciprocal"
    RSQRT = "rsqrt"
    EXP = "exp"
    PRNG = "prng"
    QUANTIZE = "quantize"
    DEQUANTIZE = "dequantize"
    REDUCE = "reduce"
    TRANSFORM = "transform"
    UNPACK = "unpack"
    REPLICATE_COLS = "replicate_cols"
    GATHER = "gather"
    SCATTER = "scatter"
    GATHER2D = "gather2d"
    SCATTER2D = "scatter2d"
    STRIDED_LOAD = "strided_load"
    STRIDED_STORE = "strided_store"
    TANH = "tanh"
    TANH_INV = "tanh_inv"
    RELU = "relu"
    RELU_INV = "relu_inv"
    SIGMOID = "sigmoid"
    SIGMOID_INV = "sigmoid_inv"
    GELU = "gelu"
    GELU_INV = "gelu_inv"
    DROPOUT = "dropout"
    DROPOUT_INV = "dropout_inv"


class BinaryKind(enum.Enum):
    ADD = "add"
    SUB = "sub"
    MUL = "mul"
    DIV = "div"
    MAX = "max"
    MIN = "min"
    MATMUL = "matmul"
    PACK = "pack"
    COMPARE = "compare"


class TernaryKind(enum.Enum):
    GEMM = "gemm"
    BRGEMM = "brgemm"
    MULADD = "muladd"
    NMULADD = "nmuladd"
    BLEND = "blend"


class CmpOp(enum.Enum):
    EQ = "eq"
    NE = "ne"
    LT = "lt"
    LE = "le"
    GT = "gt"
    GE = "ge"


class ReduceAxis(enum.Enum):
    ROWS = "rows"
    COLS = "cols"
    ALL = "all"


class ReduceOp(enum.Enum):
    SUM = "sum"
    MUL = "mul"
    MIN = "min"
    MAX = "max"


@dataclass(frozen=True)
class ReduceSpec:
    axis: ReduceAxis
    op: ReduceOp
    squared: bool = False


class TransformKind(enum.Enum):
    TRANSPOSE = "transpose"
    VNNI = "vnni"
    VNNI_TO_VNNIT = "vnni_to_vnnit"


@dataclass(frozen=True)
class TransformSpec:
    kind: TransformKind
    alpha: int = 0
    alpha_out: int = 0
    rows: int = 0
    cols: int = 0


class Approx(enum.Enum):
    PADE78 = "pade78"
    MINIMAX16 = "minimax16"
    TAYLOR2 = "taylor2"
    EXACT = "exact"


DEFAULT_APPROX = {
    UnaryKind.GELU: Approx.MINIMAX16,
    UnaryKind.GELU_INV: Approx.MINIMAX16,
    UnaryKind.EXP: Approx.TAYLOR2,
}


class InvalidSpecError(ValueError):
    """Kernel spec rejected; ``code`` is 'shape', 'dtype' or 'flag' (ops.py:174-179)."""

    def __init__(self, code: str, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code


_UNARY_CODE = {
    UnaryKind.IDENTITY: 0, UnaryKind.ZERO: 1, UnaryKind.SQUARE: 2, UnaryKind.INC: 3,
    UnaryKind.DEC: 4, UnaryKind.SQRT: 5, UnaryKind.RECIPROCAL: 6, UnaryKind.RSQRT: 7,
    UnaryKind.EXP: 8, UnaryKind.RELU: 9, UnaryKind.RELU_INV: 10, UnaryKind.GELU: 11,
    UnaryKind.GELU_INV: 12,
}
_BINARY_CODE = {BinaryKind.ADD: 0, BinaryKind.SUB: 1, BinaryKind.MUL: 2, BinaryKind.DIV: 3,
                BinaryKind.MAX: 4, BinaryKind.MIN: 5}
_OUT_OF_SCOPE = ("not on the BRGEMM hot path (SURVEY.md §2: out of scope for the sm_100a "
                 "port)")


def _require_logical_shape(v: TensorView, rows: int, cols: int, what: str) -> None:
    if (v.desc.rows, v.desc.cols) != (rows, cols):
        raise TensorError(f"{what}: expected {rows}x{cols}, got {v.desc.rows}x{v.desc.cols}")


def _join_shapes(shapes: Sequence[tuple[int, int]]) -> tuple[int, int]:
    """ops.py:260-266."""
    rows = max(s[0] for s in shapes)
    cols = max(s[1] for s in shapes)
    for r, c in shapes:
        if r not in (1, rows) or c not in (1, cols):
            raise InvalidSpecError("shape", f"cannot broadcast-join {shapes}")
    return rows, cols


def _cuda(*views):
    for v in views:
        if v is not None:
            v.require_cuda()
    return _lib.load()


# ---------------------------------------------------------------------------
# PRNG state (ops.py:195-236)
# ---------------------------------------------------------------------------

class PrngState:
    """Per-column Marsaglia xorshift128 streams (ops.py:202-236), resident on
    the GPU as uint32 [4][ncols] (x, y, z, w rows).

    Seeding is the reference's: splitmix64(seed ^ col), never all-zero.  A
    call that draws advances the streams in place (the kernel writes the
    advanced words to a second buffer and the two are swapped), so successive
    DROPOUT calls see successive uniforms exactly as the reference's do.

    Stream safety: every launch that writes the state (seeding, each draw)
    records an event on its stream, and the next draw -- on whatever stream
    it is issued -- waits for that event first, so the ping-pong buffers
    are never read before the previous writer finished.
    """

    def __init__(self, seed: int, ncols: int = 1, device=None):
        if ncols < 1:
            raise TensorError("PrngState needs ncols >= 1")
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.ncols = int(ncols)
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self._bufs = [torch.empty((4, self.ncols), dtype=torch.int32, device=dev) for _ in range(2)]
        self._cur = 0
        self._ready = None
        lib = _lib.load()
        with torch.cuda.device(dev):
            _lib.check(lib.tpp_prng_seed(C.c_uint64(self.seed), self.ncols, self._bufs[0].data_ptr(),
                                         _lib.stream_ptr(None)), "PrngState")
            self._mark(None)

    def _mark(self, stream) -> None:
        """Record that the state was last written on ``stream``.  Inside a
        CUDA-graph capture the graph's own stream order applies (an event
        recorded in a capture cannot be waited on outside it)."""
        if torch.cuda.is_current_stream_capturing():
            self._ready = None
            return
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(s)
        self._ready = ev

    def _acquire(self, stream) -> None:
        """Order ``stream`` after the last write of the state."""
        if self._ready is not None and not torch.cuda.is_current_stream_capturing():
            s = stream if stream is not None else torch.cuda.current_stream(self.device)
            s.wait_event(self._ready)

    @property
    def device(self) -> torch.device:
        return self._bufs[0].device

    def _io(self):
        return self._bufs[self._cur], self._bufs[1 - self._cur]

    def _advance(self) -> None:
        self._cur = 1 - self._cur

    def words(self) -> torch.Tensor:
        """Current stream words as a uint32-valued int64 tensor [4, ncols]."""
        self._acquire(None)
        return self._bufs[self._cur].to(torch.int64) & 0xFFFFFFFF

    def _word(self, r: int):
        return (self.words()[r].cpu().numpy()).astype("uint32")

    x = property(lambda self: self._word(0))
    y = property(lambda self: self._word(1))
    z = property(lambda self: self._word(2))
    w = property(lambda self: self._word(3))

    def uniform_block(self, rows: int) -> torch.Tensor:
        """rows x ncols FP32 uniforms in [0, 1) (ops.py:230-236), on the GPU."""
        from .tensor import alloc
        out = alloc(TensorDesc(rows, self.ncols, rows, DType.FP32), device=self.device)
        _prng_fill_state(self, out, None)
        return out.primary.view(self.ncols, rows).t()

    def step(self):
        """Advance every stream once; returns one 32-bit word per stream."""
        self.uniform_block(1)
        return self.w


def _prng_fill_state(state: PrngState, out: TensorView, stream) -> None:
    lib = _cuda(out)
    src, dst = state._io()
    state._acquire(stream)
    _lib.check(lib.tpp_prng_fill(src.data_ptr(), dst.data_ptr(), out.desc.c(), out.ptr,
                                 _lib.stream_ptr(stream)), "PRNG")
    state._advance()
    state._mark(stream)


def _prng_state_for(view: Optional[TensorView], cols: int, what: str) -> PrngState:
    state = (view.tertiary or {}).get("prng") if view is not None else None
    if state is None:
        raise InvalidSpecError("flag", f"{what} needs a PrngState in tertiary")
    if state.ncols != cols:  # ops.py:425-426 / 438-439: a fresh stream set, not persisted
        state = PrngState(state.seed, cols, device=state.device)
    return state


def _prng_fill(inp: Optional[TensorView], out: TensorView, stream=None) -> None:
    """ops.py:416-427."""
    if out.desc.dtype is not DType.FP32:
        raise InvalidSpecError("dtype", "PRNG output must be FP32")
    state = _prng_state_for(inp, out.desc.cols, "PRNG")
    _prng_fill_state(state, out, stream)


def _dropout(inp: TensorView, out: TensorView, p: Optional[float], stream=None) -> None:
    """ops.py:430-444: keep = u >= float32(p); out = keep ? x / (1 - p) : 0."""
    _require_logical_shape(out, inp.desc.rows, inp.desc.cols, f"{UnaryKind.DROPOUT} output")
    if p is None:
        raise InvalidSpecError("flag", "DROPOUT needs the drop probability p")
    if not 0.0 <= p < 1.0:
        raise InvalidSpecError("flag", f"dropout p must be in [0, 1), got {p}")
    state = _prng_state_for(inp, inp.desc.cols, "DROPOUT")
    lib = _cuda(inp, out)
    # every mask byte (padding bits included) is written by the kernel
    mask = torch.empty(bitmask_bytes(inp.desc.rows, inp.desc.cols), dtype=torch.uint8,
                       device=out.primary.device)
    src, dst = state._io()
    state._acquire(stream)
    _lib.check(lib.tpp_dropout(inp.desc.c(), inp.ptr, src.data_ptr(), dst.data_ptr(), float(p),
                               out.desc.c(), out.ptr, mask.data_ptr(), _lib.stream_ptr(stream)),
               "DROPOUT")
    state._advance()
    state._mark(stream)
    out.secondary = mask


def _dropout_inv(inp: TensorView, out: TensorView, p: Optional[float], stream=None) -> None:
    """ops.py:378-382."""
    _require_logical_shape(out, inp.desc.rows, inp.desc.cols, f"{UnaryKind.DROPOUT_INV} output")
    if p is None:
        raise InvalidSpecError("flag", "DROPOUT_INV needs the keep probability")
    if inp.secondary is None:
        raise TensorError("DROPOUT_INV requires a recorded bitmask in secondary")
    lib = _cuda(inp, out)
    _lib.check(lib.tpp_dropout_inv(inp.desc.c(), inp.ptr, inp.secondary.data_ptr(), float(p),
                                   out.desc.c(), out.ptr, _lib.stream_ptr(stream)), "DROPOUT_INV")


def _quantize(inp: TensorView, out: TensorView, stream=None) -> None:
    """ops.py:447-460: symmetric per-tensor INT8; the scale lands in
    out.tertiary['scale'] (read back to the host, as the reference's is a
    Python float)."""
    if inp.desc.dtype is not DType.FP32 or out.desc.dtype is not DType.INT8:
        raise InvalidSpecError("dtype", "QUANTIZE is FP32 -> INT8")
    _require_logical_shape(out, inp.desc.rows, inp.desc.cols, "QUANTIZE output")
    lib = _cuda(inp, out)
    scale = (inp.tertiary or {}).get("scale")
    dev = out.primary.device
    ws = torch.empty(2, dtype=torch.float64, device=dev)  # [0]: amax word, [1]: scale used
    _lib.check(lib.tpp_quantize(inp.desc.c(), inp.ptr, 0 if scale is None else 1,
                                0.0 if scale is None else float(scale), out.desc.c(), out.ptr,
                                ws.data_ptr(), ws.data_ptr() + 8, _lib.stream_ptr(stream)), "QUANTIZE")
    out.tertiary = dict(out.tertiary or {})
    out.tertiary["scale"] = float(ws[1].item())


def _dequantize(inp: TensorView, out: TensorView, stream=None) -> None:
    """ops.py:463-469."""
    if inp.desc.dtype is not DType.INT8 or out.desc.dtype is not DType.FP32:
        raise InvalidSpecError("dtype", "DEQUANTIZE is INT8 -> FP32")
    scale = (inp.tertiary or {}).get("scale")
    if scale is None:
        raise InvalidSpecError("flag", "DEQUANTIZE needs tertiary['scale']")
    _require_logical_shape(out, inp.desc.rows, inp.desc.cols, "DEQUANTIZE output")
    lib = _cuda(inp, out)
    _lib.check(lib.tpp_dequantize(inp.desc.c(), inp.ptr, float(scale), out.desc.c(), out.ptr,
                                  _lib.stream_ptr(stream)), "DEQUANTIZE")


# ---------------------------------------------------------------------------
# unary (ops.py:284-386)
# ---------------------------------------------------------------------------

def apply_unary(kind: UnaryKind, inp: Optional[TensorView], out: TensorView,
                approx_flag: Approx | None = None,
                reduce_spec: ReduceSpec | None = None,
                transform_spec: TransformSpec | None = None,
                bitmask_output: bool = False,
                dropout_p: float | None = None,
                times: int | None = None, stream=None) -> None:
    s = _lib.stream_ptr(stream) if torch.cuda.is_available() else 0
    if kind is UnaryKind.ZERO:
        lib = _cuda(out)
        _lib.check(lib.tpp_unary(_UNARY_CODE[kind], None, None, None, out.desc.c(), out.ptr,
                                 None, s), "ZERO")
        return
    if inp is None:
        raise TensorError(f"{kind} requires an input view")
    if kind is UnaryKind.REDUCE:
        if reduce_spec is None:
            raise InvalidSpecError("flag", "REDUCE needs a ReduceSpec")
        reduce(inp, reduce_spec, out, stream=stream)
        return
    if kind is UnaryKind.TRANSFORM:
        if transform_spec is None:
            raise InvalidSpecError("flag", "TRANSFORM needs a TransformSpec")
        transform(inp, transform_spec, out, stream=stream)
        return
    if kind is UnaryKind.PRNG:
        _prng_fill(inp, out, stream)
        return
    if kind is UnaryKind.QUANTIZE:
        _quantize(inp, out, stream)
        return
    if kind is UnaryKind.DEQUANTIZE:
        _dequantize(inp, out, stream)
        return
    if kind in (UnaryKind.STRIDED_LOAD, UnaryKind.STRIDED_STORE):
        raise InvalidSpecError("flag", "use strided_load/strided_store helpers")
    if kind is UnaryKind.DROPOUT:
        _dropout(inp, out, dropout_p, stream)
        return
    if kind is UnaryKind.DROPOUT_INV:
        _dropout_inv(inp, out, dropout_p, stream)
        return
    if kind not in _UNARY_CODE:
        raise NotImplementedError(f"{kind}: {_OUT_OF_SCOPE}")
    sel = approx_flag or DEFAULT_APPROX.get(kind)
    if sel is Approx.EXACT or (sel is not None and sel is not DEFAULT_APPROX.get(kind)):
        raise NotImplementedError(f"{kind} with approximation {sel}: {_OUT_OF_SCOPE}")
    _require_logical_shape(out, inp.desc.rows, inp.desc.cols, f"{kind} output")
    aux = None
    mask_out = None
    if kind is UnaryKind.RELU_INV:
        if inp.secondary is None:
            raise TensorError("RELU_INV requires a recorded bitmask in secondary")
        aux = inp.secondary
    elif kind is UnaryKind.GELU_INV:
        if inp.secondary is None:
            raise TensorError("backward kind requires the forward input in secondary")
        aux = inp.secondary
    lib = _cuda(inp, out)
    if kind is UnaryKind.RELU and bitmask_output:
        mask_out = alloc_bitmask(inp.desc.rows, inp.desc.cols, device=out.primary.device)
    rc = lib.tpp_unary(_UNARY_CODE[kind], inp.desc.c(), inp.ptr,
                       aux.data_ptr() if aux is not None else None, out.desc.c(), out.ptr,
                       mask_out.data_ptr() if mask_out is not None else None, s)
    _lib.check(rc, str(kind))
    if mask_out is not None:
        out.secondary = mask_out


def _identity(inp: TensorView, out: TensorView, stream=None) -> None:
    apply_unary(UnaryKind.IDENTITY, inp, out, stream=stream)


# ---------------------------------------------------------------------------
# reduce (ops.py:484-522)
# ---------------------------------------------------------------------------

_AXIS = {ReduceAxis.ROWS: 0, ReduceAxis.COLS: 1, ReduceAxis.ALL: 2}
_ROP = {ReduceOp.SUM: 0, ReduceOp.MUL: 1, ReduceOp.MIN: 2, ReduceOp.MAX: 3}


def reduce(inp: TensorView, spec: ReduceSpec, out: TensorView, stream=None) -> None:
    d = inp.desc
    exp_shape = {ReduceAxis.ROWS: (d.rows, 1), ReduceAxis.COLS: (1, d.cols),
                 ReduceAxis.ALL: (1, 1)}[spec.axis]
    _require_logical_shape(out, *exp_shape, what="reduce output")
    lib = _cuda(inp, out)
    _lib.check(lib.tpp_reduce(d.c(), inp.ptr, _AXIS[spec.axis], _ROP[spec.op], int(spec.squared),
                              out.desc.c(), out.ptr, _lib.stream_ptr(stream)), "reduce")


# ---------------------------------------------------------------------------
# transforms (ops.py:525-592)
# ---------------------------------------------------------------------------

def vnni_alpha_for(dtype: DType) -> int:
    if dtype.bits == 16:
        return 2
    if dtype.bits == 8:
        return 4
    raise InvalidSpecError("dtype", f"no VNNI group size for {dtype}")


def _check_alpha(dtype: DType, alpha: int) -> None:
    want = vnni_alpha_for(dtype)
    if alpha != want:
        raise InvalidSpecError("flag", f"alpha {alpha} incompatible with {dtype} (want {want})")


_TKIND = {TransformKind.TRANSPOSE: 0, TransformKind.VNNI: 1, TransformKind.VNNI_TO_VNNIT: 2}


def transform(inp: TensorView, spec: TransformSpec, out: TensorView, stream=None) -> None:
    """TRANSPOSE, VNNI formatting or VNNI -> VNNI-transpose, bit-exact."""
    d = inp.desc
    if spec.kind is TransformKind.TRANSPOSE:
        _require_logical_shape(out, d.cols, d.rows, "TRANSPOSE output")
    elif spec.kind is TransformKind.VNNI:
        _check_alpha(d.dtype, spec.alpha)
        g = -(-d.cols // spec.alpha)
        _require_logical_shape(out, d.rows * spec.alpha, g, "VNNI output")
    elif spec.kind is TransformKind.VNNI_TO_VNNIT:
        _check_alpha(d.dtype, spec.alpha)
        _check_alpha(out.desc.dtype, spec.alpha_out)
        if spec.rows <= 0 or spec.cols <= 0:
            raise InvalidSpecError("shape", "VNNI_TO_VNNIT needs the logical extent")
        g = -(-spec.rows // spec.alpha_out)
        _require_logical_shape(out, spec.cols * spec.alpha_out, g, "VNNI_TO_VNNIT output")
    else:
        raise InvalidSpecError("flag", f"unknown transform {spec.kind}")
    lib = _cuda(inp, out)
    _lib.check(lib.tpp_transform(_TKIND[spec.kind], d.c(), inp.ptr, spec.alpha, spec.alpha_out,
                                 spec.rows, spec.cols, out.desc.c(), out.ptr,
                                 _lib.stream_ptr(stream)), "transform")


# ---------------------------------------------------------------------------
# binary / ternary (ops.py:747-816)
# ---------------------------------------------------------------------------

def apply_binary(kind: BinaryKind, a: TensorView, b: TensorView, out: TensorView,
                 cmp: CmpOp | None = None, stream=None) -> None:
    if kind is BinaryKind.MATMUL:
        from . import contraction
        contraction.matmul(a, b, out)
        return
    if kind not in _BINARY_CODE:
        raise NotImplementedError(f"{kind}: {_OUT_OF_SCOPE}")
    try:
        rows, cols = _join_shapes([(a.desc.rows, a.desc.cols), (b.desc.rows, b.desc.cols)])
    except InvalidSpecError as e:
        raise TensorError(str(e)) from None
    _require_logical_shape(out, rows, cols, f"{kind} output")
    lib = _cuda(a, b, out)
    _lib.check(lib.tpp_binary(_BINARY_CODE[kind], a.desc.c(), a.ptr, b.desc.c(), b.ptr,
                              out.desc.c(), out.ptr, _lib.stream_ptr(stream)), str(kind))


def apply_ternary(kind: TernaryKind, a: TensorView, b: TensorView, c: TensorView,
                  out: TensorView, stream=None) -> None:
    if kind in (TernaryKind.GEMM, TernaryKind.BRGEMM):
        raise InvalidSpecError("flag", "GEMM/BRGEMM live in the gemm module")
    if kind is TernaryKind.BLEND:
        raise NotImplementedError(f"{kind}: {_OUT_OF_SCOPE}")
    rows, cols = _join_shapes([(a.desc.rows, a.desc.cols), (b.desc.rows, b.desc.cols),
                               (c.desc.rows, c.desc.cols)])
    _require_logical_shape(out, rows, cols, f"{kind} output")
    lib = _cuda(a, b, c, out)
    code = 0 if kind is TernaryKind.MULADD else 1
    _lib.check(lib.tpp_ternary(code, a.desc.c(), a.ptr, b.desc.c(), b.ptr, c.desc.c(), c.ptr,
                               out.desc.c(), out.ptr, _lib.stream_ptr(stream)), str(kind))


# ---------------------------------------------------------------------------
# dispatch (ops.py:823-975)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class KernelSpec:
    """A fully specified primitive instance; the output shape is a total
    function of (kind, inputs, flags)."""
    kind: UnaryKind | BinaryKind | TernaryKind
    ins: tuple
    approx: Approx | None = None
    reduce: ReduceSpec | None = None
    transform: TransformSpec | None = None
    cmp: CmpOp | None = None
    bitmask_output: bool = False
    dropout_p: float | None = None
    times: int | None = None
    index_desc: TensorDesc | None = None

    def output_desc(self) -> TensorDesc:
        return infer_output_desc(self)


def _float_join(dts) -> DType:
    if DType.FP64 in dts:
        return DType.FP64
    return DType.FP32 if all(d.is_float for d in dts) else DType.INT32


def infer_output_desc(spec: KernelSpec) -> TensorDesc:
    """Output descriptor rules of ops.py:843-938 for the hot-path kinds."""
    k, ins = spec.kind, spec.ins
    if isinstance(k, UnaryKind):
        if len(ins) != 1:
            raise InvalidSpecError("shape", "unary spec takes one input desc")
        d = ins[0]
        if k is UnaryKind.REDUCE:
            if spec.reduce is None:
                raise InvalidSpecError("flag", "REDUCE needs a ReduceSpec")
            r, c = {ReduceAxis.ROWS: (d.rows, 1), ReduceAxis.COLS: (1, d.cols),
                    ReduceAxis.ALL: (1, 1)}[spec.reduce.axis]
            return TensorDesc(r, c, r, DType.FP64 if d.dtype is DType.FP64 else DType.FP32)
        if k is UnaryKind.TRANSFORM:
            t = spec.transform
            if t is None:
                raise InvalidSpecError("flag", "TRANSFORM needs a TransformSpec")
            if t.kind is TransformKind.TRANSPOSE:
                return TensorDesc(d.cols, d.rows, d.cols, d.dtype)
            if t.kind is TransformKind.VNNI:
                g = -(-d.cols // t.alpha)
                return TensorDesc(d.rows * t.alpha, g, d.rows * t.alpha, d.dtype)
            g = -(-t.rows // t.alpha_out)
            return TensorDesc(t.cols * t.alpha_out, g, t.cols * t.alpha_out, d.dtype)
        if k is UnaryKind.DROPOUT and spec.dropout_p is None:
            raise InvalidSpecError("flag", "DROPOUT needs p")
        return TensorDesc(d.rows, d.cols, d.rows, d.dtype)
    if isinstance(k, BinaryKind):
        if len(ins) != 2:
            raise InvalidSpecError("shape", "binary spec takes two input descs")
        a, b = ins
        if k is BinaryKind.MATMUL:
            if a.cols != b.rows:
                raise InvalidSpecError("shape", f"matmul inner dims {a.cols} != {b.rows}")
            out_dt = a.dtype if a.dtype is DType.FP64 else (
                DType.INT32 if a.dtype is DType.INT8 else DType.FP32)
            return TensorDesc(a.rows, b.cols, a.rows, out_dt)
        rows, cols = _join_shapes([(a.rows, a.cols), (b.rows, b.cols)])
        if k is BinaryKind.COMPARE:
            if spec.cmp is None:
                raise InvalidSpecError("flag", "COMPARE needs a predicate")
            return TensorDesc(rows, cols, rows, DType.BIT)
        if a.dtype.is_float != b.dtype.is_float:
            raise InvalidSpecError("dtype", "mixed int/float elementwise inputs")
        out_dt = a.dtype if a.dtype == b.dtype else _float_join((a.dtype, b.dtype))
        return TensorDesc(rows, cols, rows, out_dt)
    if isinstance(k, TernaryKind):
        if len(ins) != 3:
            raise InvalidSpecError("shape", "ternary spec takes three input descs")
        a, b, c = ins
        if k in (TernaryKind.GEMM, TernaryKind.BRGEMM):
            if a.cols != b.rows or (c.rows, c.cols) != (a.rows, b.cols):
                raise InvalidSpecError("shape", "GEMM operand shapes inconsistent")
            return TensorDesc(c.rows, c.cols, c.rows, c.dtype)
        rows, cols = _join_shapes([(a.rows, a.cols), (b.rows, b.cols), (c.rows, c.cols)])
        return TensorDesc(rows, cols, rows, _float_join((a.dtype, b.dtype, c.dtype)))
    raise InvalidSpecError("flag", f"unknown kind {k}")


class Kernel:
    """An immutable, dispatched primitive instance (ops.py:941-961)."""

    __slots__ = ("spec", "out_desc")

    def __init__(self, spec: KernelSpec):
        self.spec = spec
        self.out_desc = infer_output_desc(spec)

    def __call__(self, *views: TensorView, out: TensorView, stream=None) -> None:
        s = self.spec
        k = s.kind
        if isinstance(k, UnaryKind):
            apply_unary(k, views[0] if views else None, out, approx_flag=s.approx,
                        reduce_spec=s.reduce, transform_spec=s.transform,
                        bitmask_output=s.bitmask_output, dropout_p=s.dropout_p, times=s.times,
                        stream=stream)
        elif isinstance(k, BinaryKind):
            apply_binary(k, views[0], views[1], out, cmp=s.cmp, stream=stream)
        else:
            apply_ternary(k, views[0], views[1], views[2], out, stream=stream)


_dispatch_cache: dict = {}
_dispatch_lock = threading.Lock()


def dispatch(spec: KernelSpec) -> Kernel:
    """Validate a spec and return the cached kernel (ops.py:964-975):
    lock-free lookup, locked insert."""
    hit = _dispatch_cache.get(spec)
    if hit is not None:
        return hit
    kern = Kernel(spec)
    with _dispatch_lock:
        return _dispatch_cache.setdefault(spec, kern)
