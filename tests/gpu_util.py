"""Helpers for the GPU parity tests (device upload/download of reference-layout buffers)."""

import numpy as np
import torch


def dev():
    return torch.device("cuda", torch.cuda.current_device())


def to_dev(a: np.ndarray) -> torch.Tensor:
    """Flat device tensor with the same bits/dtype as the host array
    (uint16 BF16 patterns -> torch.bfloat16)."""
    a = np.ascontiguousarray(a).reshape(-1)
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).to(dev())
    return torch.from_numpy(a.copy()).to(dev())


def to_host(t: torch.Tensor) -> np.ndarray:
    t = t.detach().contiguous()
    if t.dtype in (torch.bfloat16, torch.int16):
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def normwise(got, ref) -> float:
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    both_nan = np.isnan(got) & np.isnan(ref)
    d = np.where(both_nan, 0.0, np.abs(got - ref))
    return float(np.max(d) / max(float(np.max(np.abs(np.where(np.isnan(ref), 0, ref)))), 1e-30))


def vnni_weights(rng, Kb, Cb, bk, bc, std):
    """Random BF16 weights, logical blocks (bk x bc) packed to VNNI-2
    [Kb][Cb][bc/2][bk][2] — the reference layout (contraction.py:238-247)."""
    from oracle import tpp_oracle as O
    wl = O.fp32_to_bf16_rne(rng.normal(0, std, (Kb, Cb, bk, bc)).astype(np.float32))
    # vnni of each (bk x bc) block: [bc/2][bk][2], element (m, k) at (k//2, m, k%2)
    wv = wl.reshape(Kb, Cb, bk, bc // 2, 2).transpose(0, 1, 3, 2, 4).copy()
    return wv
