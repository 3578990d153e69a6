"""Blocked-MLP training on tcgen05 (BASELINE cfg 5): forward, softmax-CE,
backward-data / backward-weights BRGEMMs and the split-SGD update, data
parallel over the minibatch with one dW allreduce per layer.

Composition of the reference TPPs (SURVEY §0.2 row "MLP training"):
  forward    fc_forward + RELU with bitmask        (kernels.py:300-329, ops.py:363-366)
  loss       softmax per token                     (kernels.py:84-99) -> (p - onehot)/B
  backward   brgemm for dX and dW, RELU_INV        (contraction.py:261, ops.py:367-369)
  update     split_sgd_step on hi/lo FP32 masters  (kernels.py:235-251)
Weights live in the UMMA-canonical packed layout [out/64][in/64][64][64]; the
hi halves of the split FP32 master ARE the BF16 weights the GEMMs read, so no
per-step re-layout is needed (the MN-major backward operands read them in
place).
"""

from __future__ import annotations

from typing import Optional, Sequence

import torch

from . import kernels as K
from .ops import UnaryKind
from .parallel import GradSync, world

BLK = 64


def pack_logical_weight(w: torch.Tensor) -> torch.Tensor:
    """Logical [out, in] -> packed [out/64][in/64][64][64] (row o, col i)."""
    o, i = w.shape
    return w.reshape(o // BLK, BLK, i // BLK, BLK).permute(0, 2, 1, 3).contiguous().reshape(-1)


def unpack_weight(flat: torch.Tensor, o: int, i: int) -> torch.Tensor:
    return flat.reshape(o // BLK, i // BLK, BLK, BLK).permute(0, 2, 1, 3).reshape(o, i)


def split_master(w32: torch.Tensor):
    """FP32 -> (hi as bfloat16 bits, lo as int16): tensor.py:292-304 on device."""
    u = w32.contiguous().view(torch.int32)
    hi = (u >> 16).to(torch.int16).view(torch.bfloat16)
    lo = (u & 0xFFFF).to(torch.int16)
    return hi, lo


def pack_master(hi: torch.Tensor, lo: torch.Tensor) -> torch.Tensor:
    """tensor.py:307-315."""
    return ((hi.view(torch.int16).to(torch.int32) << 16) | (lo.to(torch.int32) & 0xFFFF)).view(torch.float32)


class BlockedMLP:
    """MLP dims[0] -> dims[1] -> ... -> dims[-1], ReLU between layers, no
    bias, BF16 activations / weights with FP32 split masters.  Activations are
    blocked [n_b][d/64][bn][64] (tokens x features)."""

    def __init__(self, dims: Sequence[int], tokens: int, bn: int = 64, lr: float = 0.01,
                 global_batch: Optional[int] = None, init_std: float = 0.02, seed: int = 0,
                 device=None, weights: Optional[Sequence[torch.Tensor]] = None, group=None,
                 grad_dtype: str = "fp32", reduce_fn=None, fuse_sgd: Optional[bool] = None,
                 overlap: bool = True, defer_join: bool = False):
        """``grad_dtype``: "fp32" (dW written and applied in FP32) or "bf16"
        (dW written as BF16 by the backward-weights epilogue, exchanged as
        BF16 — half the allreduce bytes — and applied by split-SGD, which
        accepts BF16 gradients like the reference's, kernels.py:235-251).
        ``reduce_fn`` replaces the dW collective (rank emulation in tests).
        ``fuse_sgd`` (default: on when there is no gradient exchange and dW is
        FP32): each layer's split-SGD runs inside its backward-weights GEMM
        epilogue, so dW is never written (``self.dw`` stays unused); results
        are bitwise those of the unfused step.
        ``overlap`` (fused-SGD steps): each hidden layer's backward-weights
        GEMM runs on a side stream, concurrently with the next layer's
        backward-data GEMM (and layer 0's with layer 1's); the tensor-core
        kernels draw their tiles dynamically, so the two fill each other's
        wave-quantisation tails.  Results are bitwise those of the serial
        order (the kernels are independent and deterministic per tile).
        ``defer_join`` (with ``overlap``): ``step()`` leaves the side stream's
        last updates in flight -- the next forward's layer-0 GEMM runs beside
        them and only its layer 1 waits (layer 0's output alternates between
        two buffers, since the in-flight dW_1 still reads the previous one).
        Call ``sync_updates()`` (or synchronize the device) before reading the
        weights or ending a timed region."""
        if grad_dtype not in ("fp32", "bf16"):
            raise ValueError("grad_dtype must be 'fp32' or 'bf16'")
        if any(d % BLK for d in dims) or tokens % bn or bn % BLK:
            raise ValueError("dims must be multiples of 64 and tokens a multiple of bn (itself a multiple of 64)")
        self.dims = list(dims)
        self.nl = len(dims) - 1
        self.tokens, self.bn, self.n_b = tokens, bn, tokens // bn
        self.lr = lr
        rank, ws = world()
        self.global_batch = global_batch or tokens * ws
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        self.hi, self.lo, self.layers = [], [], []
        for l in range(self.nl):
            o, i = dims[l + 1], dims[l]
            if weights is not None:
                w32 = weights[l].to(dev, torch.float32)
            else:
                w32 = torch.randn(o, i, generator=gen, device=dev) * init_std
            hi, lo = split_master(pack_logical_weight(w32))
            self.hi.append(hi)
            self.lo.append(lo)
            act = UnaryKind.RELU if l < self.nl - 1 else None
            self.layers.append(K.FcLayer(o // BLK, i // BLK, BLK, BLK, None, activation=act, w_packed=hi))
        # activations h[0] = input, h[l] = output of layer l-1 (BF16); masks of h[1..nl-1]
        self.h = [None] + [torch.empty(tokens * dims[l], dtype=torch.bfloat16, device=dev)
                           for l in range(1, self.nl)]
        self.mask = [None] + [torch.empty(tokens * dims[l] // 8, dtype=torch.uint8, device=dev)
                              for l in range(1, self.nl)]
        self.logits = torch.empty(tokens * dims[-1], dtype=torch.float32, device=dev)
        self.g = [torch.empty(tokens * dims[l], dtype=torch.bfloat16, device=dev) for l in range(1, self.nl + 1)]
        self.grad_dtype = grad_dtype
        dwt = torch.float32 if grad_dtype == "fp32" else torch.bfloat16
        self.dw = [torch.empty(dims[l + 1] * dims[l], dtype=dwt, device=dev) for l in range(self.nl)]
        self.loss = torch.empty(tokens, dtype=torch.float32, device=dev)
        self.sync = GradSync(group, reduce_fn=reduce_fn, device=dev)
        if fuse_sgd is None:
            fuse_sgd = not self.sync.active and grad_dtype == "fp32"
        if fuse_sgd and (self.sync.active or grad_dtype != "fp32"):
            raise ValueError("fused split-SGD needs FP32 gradients and no gradient exchange")
        self.fuse_sgd = fuse_sgd
        self.overlap = overlap and fuse_sgd
        self._side = torch.cuda.Stream(device=dev) if self.overlap else None
        self.defer_join = bool(defer_join) and self.overlap and self.nl >= 2
        self._pending = None          # event on the side stream: the deferred updates
        self._pending_captured = False
        self._h1_alt = torch.empty_like(self.h[1]) if self.defer_join else None
        # optional per-launch hook (label) called right after each main-stream
        # launch -- bench.py records CUDA events there for the step breakdown
        self.trace = None

    # ------------------------------------------------------------------
    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x: BF16 blocked [n_b][d0/64][bn][64]; returns FP32 logits (blocked)."""
        self.h[0] = x
        deferred = self._pending is not None
        if self.defer_join:   # the previous step's dW_1 may still read h[1]
            self.h[1], self._h1_alt = self._h1_alt, self.h[1]
        for l, layer in enumerate(self.layers):
            if l == 1 and self._pending is not None:
                self._join_pending()
            if l < self.nl - 1:
                layer.forward(self.h[l], self.n_b, self.bn, out=self.h[l + 1], relu_mask=self.mask[l + 1],
                              dynamic_tiles=deferred and l == 0)
            else:
                layer.forward(self.h[l], self.n_b, self.bn, out=self.logits, out_fp32=True)
            if self.trace:
                self.trace(f"fwd{l}")
        return self.logits

    def backward(self, targets: torch.Tensor) -> None:
        """Softmax-CE gradient, then per layer (last first) dW and dX with
        the ReLU mask fused.  Each layer's dW bucket is handed to the
        gradient exchange as soon as it is written (it overlaps the remaining
        backward GEMMs) and its split-SGD update as soon as the layer's
        backward-data GEMM — the last reader of its weights — is issued."""
        nl = self.nl
        tr = self.trace
        K.softmax_xent_blocked(self.logits, targets, self.n_b, self.dims[-1] // BLK, self.bn, BLK,
                               1.0 / self.global_batch, dlogits=self.g[nl - 1], loss=self.loss)
        if tr:
            tr("xent")
        if self.fuse_sgd:
            # the per-launch trace (bench breakdown) times the serial order
            main = torch.cuda.current_stream(self.device)
            side = self._side if tr is None else None
            dyn = side is not None   # the GEMMs that run side by side draw their tiles dynamically
            for l in range(nl - 1, -1, -1):
                layer = self.layers[l]
                if l > 0:   # the last reader of the layer's weights goes first
                    layer.backward_data(self.g[l], self.n_b, self.bn, relu_mask_in=self.mask[l],
                                        out=self.g[l - 1], dynamic_tiles=dyn and l < nl - 1)
                    if tr:
                        tr(f"dx{l}")
                if side is not None and l > 0:
                    # dW_l + SGD after dX_l (it rewrites W_l), beside dX_{l-1}
                    side.wait_stream(main)
                    with torch.cuda.stream(side):
                        layer.backward_weights_sgd(self.g[l], self.h[l], self.n_b, self.bn, self.lo[l], self.lr,
                                                   dynamic_tiles=True)
                else:
                    layer.backward_weights_sgd(self.g[l], self.h[l], self.n_b, self.bn, self.lo[l], self.lr,
                                               dynamic_tiles=dyn)
                if tr:
                    tr(f"dw{l}")
            if side is not None:
                if self.defer_join:
                    ev = torch.cuda.Event()
                    ev.record(side)
                    self._pending = ev
                    self._pending_captured = torch.cuda.is_current_stream_capturing()
                else:
                    main.wait_stream(side)
            return
        for l in range(nl - 1, -1, -1):
            layer = self.layers[l]
            layer.backward_weights(self.g[l], self.h[l], self.n_b, self.bn, out=self.dw[l])
            if tr:
                tr(f"dw{l}")
            self.sync.grad_ready(self.dw[l])
            if l > 0:
                layer.backward_data(self.g[l], self.n_b, self.bn, relu_mask_in=self.mask[l],
                                    out=self.g[l - 1])
                if tr:
                    tr(f"dx{l}")
            self.sync.update_ready(lambda l=l: self._update(l))

    def _update(self, l: int) -> None:
        K.split_sgd_flat(self.hi[l], self.lo[l], self.dw[l], self.lr)
        if self.trace and not self.sync.active:
            self.trace(f"sgd{l}")

    def step(self) -> None:
        """Complete the step: every layer's exchange and split-SGD update is
        ordered before whatever the caller issues next (with ``defer_join``:
        except the side stream's last updates, see ``sync_updates``)."""
        self.sync.finish()
        if not self.defer_join:
            self.sync_updates()
        if self.trace:
            self.trace("step")

    def sync_updates(self) -> None:
        """Order every deferred weight update before the caller's next work."""
        if self._pending is not None:
            self._join_pending()

    def _join_pending(self) -> None:
        if torch.cuda.is_current_stream_capturing() and not self._pending_captured:
            raise RuntimeError("BlockedMLP(defer_join=True): call sync_updates() before capturing a CUDA graph "
                               "(the capture cannot wait on the eager steps' deferred updates)")
        torch.cuda.current_stream(self.device).wait_event(self._pending)
        self._pending = None

    def train_step(self, x: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        self.forward(x)
        self.backward(targets)
        self.step()
        return self.loss

    # ------------------------------------------------------------------
    def master_weight(self, l: int) -> torch.Tensor:
        """FP32 master weight of layer l as a logical [out, in] matrix."""
        self.sync_updates()
        return unpack_weight(pack_master(self.hi[l], self.lo[l]), self.dims[l + 1], self.dims[l])

    def gemm_flops(self, label: str) -> int:
        """Algorithmic flops of the GEMM behind a trace label (fwd{l}, dw{l}, dx{l})."""
        if not (label.startswith("fwd") or label[:2] in ("dw", "dx")):
            return 0
        l = int(label[-1])
        return 2 * self.tokens * self.dims[l] * self.dims[l + 1]

    @property
    def flops_per_step(self) -> int:
        t = self.tokens
        fwd = sum(2 * t * self.dims[l] * self.dims[l + 1] for l in range(self.nl))
        dx = sum(2 * t * self.dims[l] * self.dims[l + 1] for l in range(1, self.nl))
        return 2 * fwd + dx  # fwd + dW (same as fwd) + dX (layers 2..nl)
