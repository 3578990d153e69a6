"""Composite kernels on the GPU — drop-in for kernels.py of the reference
(/root/reference/pkg/src/tensorprim/kernels.py) on the BRGEMM hot path:
``fc_forward`` (FcSpec), ``layernorm``, ``softmax``, ``split_sgd_step``;
plus the B200 layer objects the paper's drivers become on a GPU:

* ``FcLayer`` — blocked BF16 fully-connected layer: weights are re-laid out
  ONCE from VNNI-2 into UMMA-canonical K-major blocks (the paper formats
  weights into VNNI once; here into the tensor-core
  layout), then every forward is one tcgen05 BRGEMM launch with bias, ReLU
  (+bitmask) / GELU, residual and BF16 RNE narrowing fused into the epilogue.
* ``layernorm_blocked`` — the LayerNorm equation TPP on the blocked
  activation layout FC produces, bitwise to the reference.
* ``Conv2d`` — direct convolution as an offset-addressed BRGEMM over the
  taps, forward and backward-data (any R x S, stride, padding:
  fused halo kernels for stride-1 'same' shapes, the reference composition on
  the grouped tcgen05 BRGEMM otherwise) and backward-weights (fused shapes).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
import math
from typing import Optional

import torch

from . import _lib
from .dtypes import DType
from .ops import UnaryKind
from .tensor import (Bcast, TensorDesc, TensorError, TensorView, alloc, broadcast)

# ---------------------------------------------------------------------------
# fully connected (kernels.py:287-329)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class FcSpec:
    """Blocked FC: A[M_b][K_b][b_k][b_m] x B[N_b][K_b][b_n][b_k] -> C[N_b][M_b][b_n][b_m]."""
    m_b: int
    n_b: int
    k_b: int
    bm: int
    bn: int
    bk: int
    activation: Optional[UnaryKind] = None


_ACT = {None: _lib.ACT_NONE, UnaryKind.RELU: _lib.ACT_RELU, UnaryKind.GELU: _lib.ACT_GELU}


def _flat(x) -> torch.Tensor:
    if isinstance(x, TensorView):
        return x.primary
    if isinstance(x, tuple):
        buf, off = x
        buf = buf.primary if isinstance(buf, TensorView) else buf
        return buf[int(off):]
    return x


def _fc_desc(spec: FcSpec, in_dtype: DType, flags: int = 0, block_n: int = 0) -> _lib.FcDescC:
    return _lib.FcDescC(spec.m_b, spec.n_b, spec.k_b, spec.bm, spec.bn, spec.bk, in_dtype.code,
                        _ACT[spec.activation], flags, block_n)


def fc_forward(spec: FcSpec, a_buf, b_buf, c: TensorView, threads: int = 1, stream=None) -> None:
    """kernels.py:300-329 — FP32, bitwise the reference: per output block a
    stride-BRGEMM over K_b in reference order, then the activation.
    (BF16 layers use :class:`FcLayer`.)"""
    bm, bn, bk = spec.bm, spec.bn, spec.bk
    if (c.desc.rows, c.desc.cols) != (bm, spec.n_b * spec.m_b * bn) or c.desc.ld != bm:
        raise TensorError("C must be a contiguous bm x (N_b*M_b*bn) block container")
    if spec.activation not in (None, UnaryKind.RELU):
        raise NotImplementedError("FP32 fc_forward: activation must be None or RELU")
    a, b = _flat(a_buf), _flat(b_buf)
    for t, n, what in ((a, spec.m_b * spec.k_b * bk * bm, "A"), (b, spec.n_b * spec.k_b * bn * bk, "B")):
        if t.dtype != torch.float32:
            raise TensorError(f"{what} buffer must be FP32")
        if t.numel() < n:
            raise TensorError(f"{what} buffer too small: {t.numel()} < {n}")
    if c.desc.dtype is not DType.FP32:
        raise TensorError("C must be FP32")
    c.require_cuda("fc_forward")
    lib = _lib.load()
    d = _fc_desc(spec, DType.FP32)
    _lib.check(lib.tpp_fc_forward(C.byref(d), a.data_ptr(), b.data_ptr(), None, None, c.ptr, None,
                                  _lib.stream_ptr(stream)), "fc_forward")


class FcLayer:
    """BF16 blocked FC layer on tcgen05 (SURVEY §0.1 naming):

    weights VNNI ``[m_b][k_b][bk/2][bm][2]`` (out-feature blocks x in-channel
    blocks), input ``[n_b][k_b][bn][bk]``, output ``[n_b][m_b][bn][bm]``,
    bias ``[m_b*bm]`` (BF16 or FP32).  ``forward`` computes
    ``out = act(W x + bias) + residual`` with every epilogue op fused and the
    reference's FP32 op order, narrowed to BF16 with RNE.
    """

    def __init__(self, m_b: int, k_b: int, bm: int, bk: int, w_vnni: Optional[torch.Tensor],
                 bias: Optional[torch.Tensor] = None, activation: Optional[UnaryKind] = None,
                 block_n: int = 0, stream=None, w_packed: Optional[torch.Tensor] = None):
        if bias is not None and (bias.numel() < m_b * bm or bias.dtype not in (torch.bfloat16, torch.float32)):
            raise TensorError("bias must hold m_b*bm BF16/FP32 values")
        self.m_b, self.k_b, self.bm, self.bk = m_b, k_b, bm, bk
        self.activation = activation
        self.bias = bias
        self.block_n = block_n
        if w_packed is not None:
            # weights already in the K-major packed layout [m_b][k_b][bm][bk]
            # (e.g. the hi halves of split-SGD master weights)
            if w_packed.dtype != torch.bfloat16 or not w_packed.is_cuda or w_packed.numel() < m_b * k_b * bm * bk:
                raise TensorError("packed weights must be a CUDA bfloat16 [m_b][k_b][bm][bk] buffer")
            self.w_packed = w_packed
            return
        if w_vnni is None or w_vnni.dtype != torch.bfloat16 or not w_vnni.is_cuda:
            raise TensorError("FcLayer weights must be a CUDA bfloat16 VNNI buffer")
        if w_vnni.numel() < m_b * k_b * bm * bk:
            raise TensorError("weight buffer too small")
        self.w_packed = torch.empty(m_b * k_b * bm * bk, dtype=torch.bfloat16, device=w_vnni.device)
        self.repack(w_vnni, stream)

    def repack(self, w_vnni: torch.Tensor, stream=None) -> None:
        """VNNI -> K-major word transpose (tpp_fc_pack_weights)."""
        lib = _lib.load()
        d = _lib.FcDescC(self.m_b, 1, self.k_b, self.bm, 1, self.bk, _lib.BF16, 0, 0, 0)
        _lib.check(lib.tpp_fc_pack_weights(C.byref(d), w_vnni.data_ptr(), self.w_packed.data_ptr(),
                                           _lib.stream_ptr(stream)), "fc_pack_weights")

    def desc(self, n_b: int, bn: int, flags: int) -> _lib.FcDescC:
        return _lib.FcDescC(self.m_b, n_b, self.k_b, self.bm, bn, self.bk, _lib.BF16,
                            _ACT[self.activation], flags, self.block_n)

    def forward(self, x: torch.Tensor, n_b: int, bn: int, out: Optional[torch.Tensor] = None,
                residual: Optional[torch.Tensor] = None, relu_mask: Optional[torch.Tensor] = None,
                out_fp32: bool = False, stream=None, dynamic_tiles: bool = False) -> torch.Tensor:
        if x.dtype != torch.bfloat16 or not x.is_cuda:
            raise TensorError("FC input must be a CUDA bfloat16 buffer")
        if x.numel() < n_b * self.k_b * bn * self.bk:
            raise TensorError("input buffer too small")
        n_out = n_b * self.m_b * bn * self.bm
        if out is None:
            out = torch.empty(n_out, dtype=torch.float32 if out_fp32 else torch.bfloat16, device=x.device)
        if out.numel() < n_out:
            raise TensorError("output buffer too small")
        flags = _lib.FC_DYNAMIC_TILES if dynamic_tiles else 0
        if self.bias is not None:
            flags |= _lib.FC_BIAS | (_lib.FC_BIAS_FP32 if self.bias.dtype == torch.float32 else 0)
        if residual is not None:
            if residual.dtype != torch.bfloat16 or residual.numel() < n_out:
                raise TensorError("residual must be a BF16 buffer shaped like the output")
            flags |= _lib.FC_RESIDUAL
        if relu_mask is not None:
            if self.activation is not UnaryKind.RELU:
                raise TensorError("a ReLU bitmask needs RELU activation")
            if relu_mask.numel() < n_b * self.m_b * bn * ((self.bm + 7) // 8):
                raise TensorError("bitmask buffer too small")
            flags |= _lib.FC_RELU_MASK
        if out_fp32 or out.dtype == torch.float32:
            flags |= _lib.FC_OUT_FP32
        lib = _lib.load()
        d = self.desc(n_b, bn, flags)
        _lib.check(lib.tpp_fc_forward(
            C.byref(d), self.w_packed.data_ptr(), x.data_ptr(),
            self.bias.data_ptr() if self.bias is not None else None,
            residual.data_ptr() if residual is not None else None, out.data_ptr(),
            relu_mask.data_ptr() if relu_mask is not None else None,
            _lib.stream_ptr(stream)), "FcLayer.forward")
        return out

    def backward_data(self, dout: torch.Tensor, n_b: int, bn: int, relu_mask_in: Optional[torch.Tensor] = None,
                      out: Optional[torch.Tensor] = None, stream=None, dynamic_tiles: bool = False) -> torch.Tensor:
        """din = dout . W  ([n_b][k_b][bn][bk], BF16), optionally masked by the
        forward input's ReLU bitmask (RELU_INV fused in the epilogue).
        ``dynamic_tiles``: tiles drawn dynamically (TPP_FC_DYNAMIC_TILES), for
        a GEMM that runs beside another one on a second stream."""
        if dout.dtype != torch.bfloat16 or dout.numel() < n_b * self.m_b * bn * self.bm:
            raise TensorError("dout must be a BF16 [n_b][m_b][bn][bm] buffer")
        n_in = n_b * self.k_b * bn * self.bk
        if out is None:
            out = torch.empty(n_in, dtype=torch.bfloat16, device=dout.device)
        flags = _lib.FC_DYNAMIC_TILES if dynamic_tiles else 0
        if relu_mask_in is not None:
            if relu_mask_in.numel() < n_b * self.k_b * bn * ((self.bk + 7) // 8):
                raise TensorError("bitmask buffer too small")
            flags |= _lib.FC_RELU_INV
        lib = _lib.load()
        d = _lib.FcDescC(self.m_b, n_b, self.k_b, self.bm, bn, self.bk, _lib.BF16, _lib.ACT_NONE, flags,
                         self.block_n)
        _lib.check(lib.tpp_fc_backward_data(
            C.byref(d), self.w_packed.data_ptr(), dout.data_ptr(),
            relu_mask_in.data_ptr() if relu_mask_in is not None else None, out.data_ptr(),
            _lib.stream_ptr(stream)), "FcLayer.backward_data")
        return out

    def backward_weights(self, dout: torch.Tensor, x: torch.Tensor, n_b: int, bn: int,
                         out: Optional[torch.Tensor] = None, fp32: bool = True, stream=None) -> torch.Tensor:
        """dW = sum over tokens of dout^T x, in the packed weight layout
        [m_b][k_b][bm][bk] (FP32 by default)."""
        if dout.dtype != torch.bfloat16 or x.dtype != torch.bfloat16:
            raise TensorError("dout and x must be BF16")
        n_w = self.m_b * self.k_b * self.bm * self.bk
        if out is None:
            out = torch.empty(n_w, dtype=torch.float32 if fp32 else torch.bfloat16, device=dout.device)
        lib = _lib.load()
        d = _lib.FcDescC(self.m_b, n_b, self.k_b, self.bm, bn, self.bk, _lib.BF16, _lib.ACT_NONE,
                         _lib.FC_OUT_FP32 if out.dtype == torch.float32 else 0, self.block_n)
        _lib.check(lib.tpp_fc_backward_weights(C.byref(d), dout.data_ptr(), x.data_ptr(), out.data_ptr(),
                                               _lib.stream_ptr(stream)), "FcLayer.backward_weights")
        return out


    def backward_weights_sgd(self, dout: torch.Tensor, x: torch.Tensor, n_b: int, bn: int, w_lo: torch.Tensor,
                             lr: float, stream=None, dynamic_tiles: bool = False) -> None:
        """dW = sum over tokens of dout^T x applied at once as split-SGD on the
        FP32 master whose hi halves are this layer's packed weights
        (``w_packed``) and lo halves ``w_lo`` (kernels.py:235-251): the FP32
        dW never leaves the chip.  Bitwise equal to ``backward_weights`` +
        ``split_sgd_flat``.  Issue the layer's backward-data first: it reads
        the weights this call updates."""
        if dout.dtype != torch.bfloat16 or x.dtype != torch.bfloat16:
            raise TensorError("dout and x must be BF16")
        n_w = self.m_b * self.k_b * self.bm * self.bk
        if w_lo.numel() < n_w or w_lo.element_size() != 2:
            raise TensorError("w_lo must hold the 16-bit lo halves of every weight")
        lib = _lib.load()
        d = _lib.FcDescC(self.m_b, n_b, self.k_b, self.bm, bn, self.bk, _lib.BF16, _lib.ACT_NONE,
                         _lib.FC_DYNAMIC_TILES if dynamic_tiles else 0, self.block_n)
        _lib.check(lib.tpp_fc_backward_weights_sgd(C.byref(d), dout.data_ptr(), x.data_ptr(),
                                                   self.w_packed.data_ptr(), w_lo.data_ptr(), float(lr),
                                                   _lib.stream_ptr(stream)), "FcLayer.backward_weights_sgd")


def softmax_xent_blocked(logits: torch.Tensor, targets: torch.Tensor, n_b: int, m_b: int, bn: int,
                         bm: int, scale: float, dlogits: Optional[torch.Tensor] = None,
                         loss: Optional[torch.Tensor] = None, stream=None):
    """Softmax cross-entropy gradient on blocked FP32 logits (tokens x
    classes): the reference softmax per token, dlogits = (p - onehot) * scale
    as BF16 in the same blocked layout; per-token loss -log p[target]."""
    if logits.dtype != torch.float32 or targets.dtype != torch.int32:
        raise TensorError("logits must be FP32 and targets int32")
    n = n_b * m_b * bn * bm
    if dlogits is None:
        dlogits = torch.empty(n, dtype=torch.bfloat16, device=logits.device)
    if loss is None:
        loss = torch.empty(n_b * bn, dtype=torch.float32, device=logits.device)
    lib = _lib.load()
    _lib.check(lib.tpp_softmax_xent_blocked(n_b, m_b, bn, bm, logits.data_ptr(), targets.data_ptr(),
                                            float(scale), dlogits.data_ptr(), loss.data_ptr(),
                                            _lib.stream_ptr(stream)), "softmax_xent_blocked")
    return dlogits, loss


# ---------------------------------------------------------------------------
# normalisation (kernels.py:106-176)
# ---------------------------------------------------------------------------


def layernorm(x: TensorView, g: TensorView, b: TensorView, eps: float, out: TensorView,
              mean_out: TensorView | None = None, var_out: TensorView | None = None,
              stream=None) -> None:
    """kernels.py:134-176 — per-row layer normalisation of a column-major
    rows x cols view, bitwise the reference (FP32 ascending sums, float64
    glue, two cascaded MULADDs)."""
    rows, cols = x.desc.rows, x.desc.cols
    if cols < 2:
        raise TensorError("layernorm needs a feature dimension of at least 2")
    if eps <= 0:
        raise TensorError("eps must be positive")
    for v, name in ((g, "G"), (b, "B")):
        if (v.desc.rows, v.desc.cols) != (rows, cols):
            raise TensorError(f"{name} must broadcast to the input shape")
    for v, name in ((mean_out, "mean"), (var_out, "var")):
        if v is not None and (v.desc.dtype is not DType.FP32 or v.desc.rows != rows
                              or v.desc.ld != rows and v.desc.cols > 1):
            raise TensorError(f"{name} output must be an FP32 rows x 1 view")
    for v in (x, g, b, out):
        v.require_cuda("layernorm")
    lib = _lib.load()
    _lib.check(lib.tpp_layernorm(x.desc.c(), x.ptr, g.desc.c(), g.ptr, b.desc.c(), b.ptr,
                                 float(eps), out.desc.c(), out.ptr,
                                 mean_out.ptr if mean_out is not None else None,
                                 var_out.ptr if var_out is not None else None,
                                 _lib.stream_ptr(stream)), "layernorm")


def layernorm_blocked(x: torch.Tensor, n_b: int, m_b: int, bn: int, bm: int, eps: float = 1e-5,
                      gamma: Optional[torch.Tensor] = None, beta: Optional[torch.Tensor] = None,
                      out: Optional[torch.Tensor] = None, mean_out: Optional[torch.Tensor] = None,
                      var_out: Optional[torch.Tensor] = None, stream=None, exact: bool = True) -> torch.Tensor:
    """LayerNorm of every token of a blocked [n_b][m_b][bn][bm] activation
    over its m_b*bm features (ascending feature order), gamma/beta FP32
    [m_b*bm] (default 1 / 0, still applied as MULADD so signed zeros match).
    ``exact=False`` selects the tolerance mode (BF16 blocked layout): tree-
    ordered statistics and FMA-contracted scaling, within 1e-5 relative of the
    exact statistics; everything else is the reference order."""
    if x.dtype not in (torch.bfloat16, torch.float32) or not x.is_cuda:
        raise TensorError("x must be a CUDA bf16/fp32 buffer")
    n = n_b * m_b * bn * bm
    if x.numel() < n:
        raise TensorError("x buffer too small")
    if out is None:
        out = torch.empty(n, dtype=x.dtype, device=x.device)
    for t, name in ((gamma, "gamma"), (beta, "beta")):
        if t is not None and (t.dtype != torch.float32 or t.numel() < m_b * bm):
            raise TensorError(f"{name} must be FP32 [m_b*bm]")
    lib = _lib.load()
    dt = _lib.BF16 if x.dtype == torch.bfloat16 else _lib.FP32
    p = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    _lib.check(lib.tpp_layernorm_blocked_ex(n_b, m_b, bn, bm, dt, x.data_ptr(), p(gamma), p(beta),
                                            float(eps), out.data_ptr(), p(mean_out), p(var_out),
                                            1 if exact else 0, _lib.stream_ptr(stream)), "layernorm_blocked")
    return out


# ---------------------------------------------------------------------------
# softmax (kernels.py:49-99)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class SoftmaxSpec:
    s1: int
    s2: int
    s3: int


def softmax(spec: SoftmaxSpec, x: TensorView, y: TensorView, strategy=None, stream=None) -> None:
    """Slice-wise softmax with exp_taylor, bitwise the reference."""
    if (x.desc.rows, x.desc.cols) != (spec.s1, spec.s2 * spec.s3):
        raise TensorError("softmax input must be s1 x (s2*s3)")
    if (y.desc.rows, y.desc.cols) != (x.desc.rows, x.desc.cols):
        raise TensorError("softmax output shape mismatch")
    x.require_cuda("softmax")
    lib = _lib.load()
    _lib.check(lib.tpp_softmax(spec.s1, spec.s2, spec.s3, x.desc.c(), x.ptr, y.desc.c(), y.ptr,
                               _lib.stream_ptr(stream)), "softmax")


# ---------------------------------------------------------------------------
# split SGD (kernels.py:235-251)
# ---------------------------------------------------------------------------


def split_sgd_step(weights, grad: TensorView, lr: float, stream=None) -> None:
    """One SGD step on hi/lo split FP32 weights: bitwise FP32 SGD."""
    from .tensor import SplitTensor
    if not isinstance(weights, SplitTensor):
        raise TensorError("weights must be a SplitTensor")
    rows, cols = weights.rows, weights.cols
    if (grad.desc.rows, grad.desc.cols) != (rows, cols):
        raise TensorError("gradient shape mismatch")
    for v in (weights.hi, weights.lo, grad):
        if v.desc.ld != rows or v.desc.bcast is not Bcast.NONE:
            raise TensorError("split_sgd_step needs contiguous views")
    if grad.desc.dtype not in (DType.FP32, DType.BF16):
        raise TensorError("gradient must be FP32 or BF16")
    grad.require_cuda("split_sgd_step")
    lib = _lib.load()
    _lib.check(lib.tpp_split_sgd(rows * cols, weights.hi.ptr, weights.lo.ptr, grad.ptr,
                                 grad.desc.dtype.code, float(lr), _lib.stream_ptr(stream)),
               "split_sgd_step")


def split_sgd_flat(hi: torch.Tensor, lo: torch.Tensor, grad: torch.Tensor, lr: float,
                   stream=None) -> None:
    """split_sgd_step on flat buffers (hi: bf16, lo: int16, grad: fp32/bf16)."""
    lib = _lib.load()
    gd = _lib.BF16 if grad.dtype == torch.bfloat16 else _lib.FP32
    _lib.check(lib.tpp_split_sgd(hi.numel(), hi.data_ptr(), lo.data_ptr(), grad.data_ptr(), gd,
                                 float(lr), _lib.stream_ptr(stream)), "split_sgd")


# ---------------------------------------------------------------------------
# direct convolution via offset BRGEMM
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class ConvSpec:
    """Direct 2-D convolution on blocked BF16 activations: input
    [N][C_b][H][W][bc], weights VNNI [K_b][C_b][R][S][bc/2][bk][2], output
    [N][K_b][P][Q][bk] with P = (H + 2 pad - R) // stride + 1 (Q likewise).
    ``stride`` = 1 and 'same' padding (2 pad = R - 1 = S - 1) with W <= 64 run
    the fused tcgen05 halo kernel; every other shape runs the reference's own
    formulation on the tensor cores: an explicitly zero-padded input and one
    OFFSET-addressed BRGEMM batch over the (r, s, c_b) taps per output row
    (K11, one grouped launch for all rows), FP32 accumulation,
    then BF16 RNE."""
    n: int
    c_b: int
    k_b: int
    h: int
    w: int
    r: int = 3
    s: int = 3
    pad: int = 1
    bc: int = 64
    bk: int = 64
    stride: int = 1

    def __post_init__(self):
        if min(self.n, self.c_b, self.k_b, self.h, self.w, self.r, self.s, self.stride) < 1 or self.pad < 0:
            raise TensorError("conv extents must be positive (pad >= 0)")
        if self.h + 2 * self.pad < self.r or self.w + 2 * self.pad < self.s:
            raise TensorError("the filter is larger than the padded input")

    def c(self) -> _lib.ConvDescC:
        return _lib.ConvDescC(self.n, self.c_b, self.k_b, self.h, self.w, self.r, self.s, self.pad,
                              self.bc, self.bk, 0, 0)

    @property
    def p(self) -> int:
        return (self.h + 2 * self.pad - self.r) // self.stride + 1

    @property
    def q(self) -> int:
        return (self.w + 2 * self.pad - self.s) // self.stride + 1

    @property
    def fused(self) -> bool:
        """The shapes the fused halo kernels (K2 forward / backward-data, K7
        backward-weights) take; the rest run the offset-BRGEMM composition."""
        return (self.stride == 1 and 2 * self.pad == self.r - 1 and 2 * self.pad == self.s - 1
                and self.w <= 64 and self.bc == 64 and self.bk == 64)

    @property
    def flops(self) -> int:
        return 2 * self.n * self.p * self.q * self.c_b * self.bc * self.k_b * self.bk * self.r * self.s


# TPP_CONV_FP32_TAIL=1: the generic conv writes FP32 accumulators and narrows
# them in a separate tpp_convert pass (the reference's two steps; A/B)
_CONV_FP32_TAIL = bool(os.environ.get("TPP_CONV_FP32_TAIL"))


class _OffsetConv:
    """One offset-BRGEMM convolution (the reference composition) on the
    tensor cores.  Batch entries = taps (r, s) x input channel blocks cb, in
    that order; A = the VNNI weight block (kb, cb, r, s); B = a bc x n slice
    of the padded input with column stride stride*bc (ldb).  A C block covers
    RB whole output rows in the padded-width position space: virtual column
    v = row * Wp + ow reads padded pixel (row*stride + r, ow*stride + s) at
    element stride*bc*v from the tap's base, uniformly across row ends, so one
    block of n = RB*Wp <= 256 columns (RB the largest divisor of P that fits)
    is one BRGEMM; the Wp - Q columns past each row's end are computed and
    dropped by the strided FP32 -> BF16 RNE pass.  Index arrays are built once
    and live on the device."""

    def __init__(self, n, ci_b, co_b, hp, wp, p, q, r, s, stride, device):
        import numpy as np
        from .contraction import ALayout, GemmSpec
        blk = 64 * 64
        rb = max(d for d in range(1, p + 1) if p % d == 0 and (d * wp <= 256 or d == 1))
        ncols = rb * wp
        self.p, self.q, self.wp, self.rows_per_block = p, q, wp, rb
        self.groups = n * co_b * (p // rb)
        self.count = r * s * ci_b
        self.spec = GemmSpec(64, ncols, 64, 64, stride * 64, 64, in_dtype=DType.BF16, out_dtype=DType.FP32,
                             a_layout=ALayout.VNNI, beta=0.0)
        nn, kb, ob = np.meshgrid(np.arange(n), np.arange(co_b), np.arange(p // rb), indexing="ij")
        rr, ss, cb = np.meshgrid(np.arange(r), np.arange(s), np.arange(ci_b), indexing="ij")
        rr, ss, cb = rr.reshape(-1), ss.reshape(-1), cb.reshape(-1)
        kbg, ng, obg = kb.reshape(-1, 1), nn.reshape(-1, 1), ob.reshape(-1, 1)
        a_off = ((kbg * ci_b + cb) * (r * s) + rr * s + ss) * blk
        # rows of the padded input the blocks reach (virtual columns past the
        # last row's end read on into the following rows): the caller pads to it
        self.rows_needed = int(((p // rb - 1) * rb * stride + (r - 1)) + ((ncols - 1) * stride + (s - 1)) // wp + 1)
        self.hp = max(hp, self.rows_needed)
        b_off = ((ng * ci_b + cb) * self.hp + obg * rb * stride + rr) * (wp * 64) + ss * 64
        c_off = ((nn * co_b + kb) * p + ob * rb).reshape(-1) * (wp * 64)
        # the grouped kernel trusts its indices: every block inside its buffer
        last = b_off + (ncols - 1) * stride * 64 + 64
        if (a_off.min() < 0 or a_off.max() + blk > co_b * ci_b * r * s * blk or b_off.min() < 0
                or last.max() > n * ci_b * self.hp * wp * 64):
            raise TensorError("conv offset plan out of bounds (internal)")
        self.a_idx = torch.from_numpy(np.ascontiguousarray(a_off.reshape(-1), dtype=np.int64)).to(device)
        self.b_idx = torch.from_numpy(np.ascontiguousarray(b_off.reshape(-1), dtype=np.int64)).to(device)
        self.c_off = torch.from_numpy(np.ascontiguousarray(c_off, dtype=np.int64)).to(device)
        # the same blocks in the BF16 output [planes][P][Q*64] (the fused
        # epilogue drops the Wp - Q columns past each row's end)
        self.c_off16 = torch.from_numpy(np.ascontiguousarray(c_off // wp * q, dtype=np.int64)).to(device)
        self.planes = n * co_b
        self.acc_elems = n * co_b * p * wp * 64
        # output-channel blocks share B lists, output rows share A lists: pairs
        # of channel blocks tile together (M = 128 MMAs) when there are two
        from .contraction import _gang_table
        self.gang = None
        if torch.device(device).type == "cuda":
            self.gang = _gang_table([int(v) for v in kbg.reshape(-1)],
                                    [(int(a), int(b)) for a, b in zip(ng.reshape(-1), obg.reshape(-1))],
                                    64, ncols, device, int(_lib.load().tpp_device_sm_count()))

    def run(self, w_vnni: torch.Tensor, xpad: torch.Tensor, out_bf16: torch.Tensor, stream=None) -> None:
        lib = _lib.load()
        d = self.spec.c()
        d.engine = _lib.ENGINE_TENSOR
        s = _lib.stream_ptr(stream)
        if not _CONV_FP32_TAIL:
            # FP32 accumulators narrowed RNE in the BRGEMM epilogue, straight
            # into the BF16 output (the same bits as the FP32 call + convert)
            table, ngangs, gm, gn = self.gang if self.gang is not None else (None, 0, 1, 1)
            _lib.check(lib.tpp_brgemm_grouped_bf16(C.byref(d), 1, w_vnni.data_ptr(), xpad.data_ptr(), 0, 0,
                                                   self.a_idx.data_ptr(), self.b_idx.data_ptr(), self.count,
                                                   out_bf16.data_ptr(), self.c_off16.data_ptr(), self.groups,
                                                   table.data_ptr() if table is not None else None, ngangs, gm, gn,
                                                   self.wp, self.q, s), "conv (offset BRGEMM, BF16 out)")
            return
        acc = torch.empty(self.acc_elems, dtype=torch.float32, device=xpad.device)
        if self.gang is not None:
            table, ngangs, gm, gn = self.gang
            _lib.check(lib.tpp_brgemm_grouped_gang(C.byref(d), 1, w_vnni.data_ptr(), xpad.data_ptr(), 0, 0,
                                                   self.a_idx.data_ptr(), self.b_idx.data_ptr(), self.count,
                                                   acc.data_ptr(), self.c_off.data_ptr(), self.groups,
                                                   table.data_ptr(), ngangs, gm, gn, s), "conv (offset BRGEMM)")
        else:
            _lib.check(lib.tpp_brgemm_grouped(C.byref(d), 1, w_vnni.data_ptr(), xpad.data_ptr(), 0, 0,
                                              self.a_idx.data_ptr(), self.b_idx.data_ptr(), self.count,
                                              acc.data_ptr(), self.c_off.data_ptr(), self.groups, s),
                       "conv (offset BRGEMM)")
        # FP32 accumulators -> BF16 RNE (dtypes.py:82-97), dropping the
        # columns past each row's end: rows = Q*64 valid elements of a padded-
        # width row (ld Wp*64), one column per output row
        cols = self.planes * self.p
        din = _lib.TensorDescC(self.q * 64, cols, self.wp * 64, DType.FP32.code, 0)
        dout = _lib.TensorDescC(self.q * 64, cols, self.q * 64, DType.BF16.code, 0)
        _lib.check(lib.tpp_convert(C.byref(din), acc.data_ptr(), C.byref(dout), out_bf16.data_ptr(), s),
                   "conv (RNE)")


def _conv_pad(x: torch.Tensor, n, cb, hi, wi, ho, wo, top, left, dil, stream=None) -> torch.Tensor:
    out = torch.empty(n * cb * ho * wo * 64, dtype=torch.bfloat16, device=x.device)
    _lib.check(_lib.load().tpp_conv_pad(n, cb, hi, wi, ho, wo, top, left, dil, x.data_ptr(), out.data_ptr(),
                                        _lib.stream_ptr(stream)), "conv_pad")
    return out


class Conv2d:
    """Weights packed once for forward ([K_b][R][S][C_b][bk][bc], K-major
    per tap) and for backward-data (taps flipped, C/K swapped); shapes outside
    the fused kernels keep the VNNI weights (forward) and the flipped,
    transposed VNNI weights (backward-data) as offset-BRGEMM A blocks."""

    def __init__(self, spec: ConvSpec, w_vnni: torch.Tensor, stream=None):
        if w_vnni.dtype != torch.bfloat16 or not w_vnni.is_cuda:
            raise TensorError("conv weights must be a CUDA bfloat16 VNNI buffer")
        need = spec.k_b * spec.c_b * spec.r * spec.s * spec.bc * spec.bk
        if w_vnni.numel() < need:
            raise TensorError("weight buffer too small")
        if spec.bc != 64 or spec.bk != 64:
            raise NotImplementedError("tensor-core conv needs bc = bk = 64")
        self.spec = spec
        lib = _lib.load()
        d = spec.c()
        s = _lib.stream_ptr(stream)
        if spec.fused:
            self.w_fwd = torch.empty(need, dtype=torch.bfloat16, device=w_vnni.device)
            self.w_bwd = torch.empty(need, dtype=torch.bfloat16, device=w_vnni.device)
            _lib.check(lib.tpp_conv_pack_weights(C.byref(d), w_vnni.data_ptr(), self.w_fwd.data_ptr(), 0, s),
                       "conv_pack_weights")
            _lib.check(lib.tpp_conv_pack_weights(C.byref(d), w_vnni.data_ptr(), self.w_bwd.data_ptr(), 1, s),
                       "conv_pack_weights(bwd)")
        else:
            self.w_vnni = w_vnni[:need].clone()
            self.w_bwd_vnni = torch.empty(need, dtype=torch.bfloat16, device=w_vnni.device)
            _lib.check(lib.tpp_conv_pack_weights(C.byref(d), w_vnni.data_ptr(), self.w_bwd_vnni.data_ptr(), 2, s),
                       "conv_pack_weights(bwd, VNNI)")
            self._fwd_plan = None
            self._bwd_plan = None

    def forward(self, x: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        sp = self.spec
        n_in = sp.n * sp.c_b * sp.h * sp.w * sp.bc
        n_out = sp.n * sp.k_b * sp.p * sp.q * sp.bk
        if x.dtype != torch.bfloat16 or x.numel() < n_in:
            raise TensorError("conv input must be a bf16 [N][C_b][H][W][bc] buffer")
        if out is None:
            out = torch.empty(n_out, dtype=torch.bfloat16, device=x.device)
        elif out.dtype != torch.bfloat16 or out.numel() < n_out:
            raise TensorError("conv output must be a bf16 [N][K_b][P][Q][bk] buffer")
        lib = _lib.load()
        if sp.fused:
            d = sp.c()
            _lib.check(lib.tpp_conv_forward(C.byref(d), self.w_fwd.data_ptr(), x.data_ptr(),
                                            out.data_ptr(), _lib.stream_ptr(stream)), "conv_forward")
            return out
        hp, wp = sp.h + 2 * sp.pad, sp.w + 2 * sp.pad
        if self._fwd_plan is None:
            self._fwd_plan = _OffsetConv(sp.n, sp.c_b, sp.k_b, hp, wp, sp.p, sp.q, sp.r, sp.s, sp.stride, x.device)
        xp = _conv_pad(x, sp.n, sp.c_b, sp.h, sp.w, self._fwd_plan.hp, wp, sp.pad, sp.pad, 1, stream)
        self._fwd_plan.run(self.w_vnni, xp, out, stream)
        return out

    def backward_data(self, dout: torch.Tensor, din: Optional[torch.Tensor] = None,
                      stream=None) -> torch.Tensor:
        """dI = the forward conv's adjoint: for stride s, dO zero-inserted
        (s - 1 zeros between pixels) and padded by R - 1 - pad (plus the rows /
        columns the forward's floor division dropped), convolved at stride 1
        with the flipped, C/K-swapped weights."""
        sp = self.spec
        n_in = sp.n * sp.c_b * sp.h * sp.w * sp.bc
        n_out = sp.n * sp.k_b * sp.p * sp.q * sp.bk
        if dout.dtype != torch.bfloat16 or dout.numel() < n_out:
            raise TensorError("dO must be a bf16 [N][K_b][P][Q][bk] buffer")
        if din is None:
            din = torch.empty(n_in, dtype=torch.bfloat16, device=dout.device)
        elif din.dtype != torch.bfloat16 or din.numel() < n_in:
            raise TensorError("dI must be a bf16 [N][C_b][H][W][bc] buffer")
        lib = _lib.load()
        if sp.fused:
            d = sp.c()
            _lib.check(lib.tpp_conv_backward_data(C.byref(d), self.w_bwd.data_ptr(), dout.data_ptr(),
                                                  din.data_ptr(), _lib.stream_ptr(stream)),
                       "conv_backward_data")
            return din
        if sp.pad > sp.r - 1 or sp.pad > sp.s - 1:
            raise NotImplementedError("conv backward-data with pad > R - 1 (the adjoint crops its input)")
        # dI[h][w] = sum_{r', s'} Zp[h + r'][w + s'] Wflip[r'][s'] with Zp the
        # zero-inserted dO shifted by R - 1 - pad: a stride-1 'valid' conv of
        # H x W outputs over an (H + R - 1) x (W + S - 1) buffer
        top, left = sp.r - 1 - sp.pad, sp.s - 1 - sp.pad
        hz, wz = sp.h + sp.r - 1, sp.w + sp.s - 1
        if self._bwd_plan is None:
            self._bwd_plan = _OffsetConv(sp.n, sp.k_b, sp.c_b, hz, wz, sp.h, sp.w, sp.r, sp.s, 1, dout.device)
        dz = _conv_pad(dout, sp.n, sp.k_b, sp.p, sp.q, self._bwd_plan.hp, wz, top, left, sp.stride, stream)
        self._bwd_plan.run(self.w_bwd_vnni, dz, din, stream)
        return din

    def backward_weights(self, x: torch.Tensor, dout: torch.Tensor, dw: Optional[torch.Tensor] = None,
                         stream=None) -> torch.Tensor:
        """dW FP32 [K_b][C_b][R][S][bc][bk] = sum over images and pixels of
        dO x shifted input.  One tcgen05 pass: every CTA keeps
        all taps' partial sums in TMEM over its rows; a second kernel adds the
        per-CTA partials in a fixed order."""
        sp = self.spec
        if not sp.fused:
            raise NotImplementedError("conv backward-weights runs the fused kernel only (stride 1, 'same' "
                                      "padding, W <= 64)")
        n_in = sp.n * sp.c_b * sp.h * sp.w * sp.bc
        n_out = sp.n * sp.k_b * sp.h * sp.w * sp.bk
        if x.dtype != torch.bfloat16 or x.numel() < n_in:
            raise TensorError("conv input must be a bf16 [N][C_b][H][W][bc] buffer")
        if dout.dtype != torch.bfloat16 or dout.numel() < n_out:
            raise TensorError("dO must be a bf16 [N][K_b][H][W][bk] buffer")
        n_w = sp.k_b * sp.c_b * sp.r * sp.s * sp.bc * sp.bk
        if dw is None:
            dw = torch.empty(n_w, dtype=torch.float32, device=x.device)
        elif dw.dtype != torch.float32 or dw.numel() < n_w:
            raise TensorError("dW must be an FP32 [K_b][C_b][R][S][bc][bk] buffer")
        lib = _lib.load()
        d = sp.c()
        ws = getattr(self, "_dw_ws", None)
        need = int(lib.tpp_conv_backward_weights_workspace_bytes(C.byref(d)))
        if need < 0:
            raise TensorError("invalid conv descriptor for backward-weights")
        if ws is None or ws.numel() * 4 < need:
            ws = torch.empty((need + 3) // 4, dtype=torch.float32, device=x.device)
            self._dw_ws = ws
        _lib.check(lib.tpp_conv_backward_weights(C.byref(d), x.data_ptr(), dout.data_ptr(), dw.data_ptr(),
                                                 ws.data_ptr(), _lib.stream_ptr(stream)), "conv_backward_weights")
        return dw


# ---------------------------------------------------------------------------
# 1-D dilated convolution (kernels.py:336-378): the address-based BRGEMM user
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class DilatedConvSpec:
    """kernels.py:336-348."""
    in_channels: int     # C
    out_channels: int    # K
    width: int           # W (input positions)
    out_width: int       # Q (output positions)
    taps: int            # S (filter size)
    dilation: int        # d
    block_q: int = 8     # output-position block (the reference's loop; results do not depend on it)

    def __post_init__(self):
        if self.out_width + (self.taps - 1) * self.dilation > self.width:
            raise TensorError("output width exceeds the dilated receptive field")


def dilated_conv1d_forward(spec: DilatedConvSpec, inp: TensorView, weights: TensorView,
                           out: TensorView, stream=None) -> None:
    """kernels.py:350-378.  ``inp`` is C x W (one column per position),
    ``weights`` (C*S) x K with row s*C + c holding tap s of channel c, ``out``
    K x Q.  The weights are transposed once (TRANSPOSE TPP), then the whole
    output is ONE batch-reduce over the S taps: A_s = W^T columns [s*C, s*C+C),
    B_s = the input columns starting at s*d.  Per output element that is the
    reference's order (taps outer, channels inner, no FMA), so the result is
    bitwise the reference's for every block_q — on the ordered BRGEMM kernel."""
    from .contraction import BrgemmBatch, GemmSpec, brgemm
    from .ops import TransformKind, TransformSpec, transform
    c_ch, k_ch, s_taps, d = spec.in_channels, spec.out_channels, spec.taps, spec.dilation
    if (inp.desc.rows, inp.desc.cols) != (c_ch, spec.width):
        raise TensorError("input must be C x W")
    if (weights.desc.rows, weights.desc.cols) != (c_ch * s_taps, k_ch):
        raise TensorError("weights must be (C*S) x K")
    if (out.desc.rows, out.desc.cols) != (k_ch, spec.out_width):
        raise TensorError("output must be K x Q")
    wt = alloc(TensorDesc(k_ch, c_ch * s_taps, k_ch, weights.desc.dtype), device=weights.primary.device)
    transform(weights, TransformSpec(TransformKind.TRANSPOSE), wt, stream=stream)
    gspec = GemmSpec(m=k_ch, n=spec.out_width, k=c_ch, lda=k_ch, ldb=inp.desc.ld, ldc=out.desc.ld,
                     in_dtype=wt.desc.dtype, out_dtype=out.desc.dtype, beta=0.0)
    batch = BrgemmBatch.stride(wt.primary, inp.primary, c_ch * k_ch, d * inp.desc.ld, s_taps)
    brgemm(gspec, batch, out, stream=stream)
