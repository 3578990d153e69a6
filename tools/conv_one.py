"""cfg 4 conv forward (N=256, 56x56, C=K=64, 3x3), a few launches, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05755_b200 as tpp  # noqa: E402

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
spec = tpp.ConvSpec(256, 1, 1, 56, 56)
xin = torch.rand(256 * 56 * 56 * 64, generator=gen, device=dev).to(torch.bfloat16)
wl = (torch.randn(1, 1, 3, 3, 64, 64, generator=gen, device=dev) * (2 / 576) ** 0.5).to(torch.bfloat16)
wv = wl.reshape(1, 1, 3, 3, 64, 32, 2).permute(0, 1, 2, 3, 5, 4, 6).contiguous().reshape(-1)
conv = tpp.Conv2d(spec, wv)
yo = torch.empty_like(xin)
for _ in range(4):
    conv.forward(xin, out=yo)
torch.cuda.synchronize()
print("ok")
