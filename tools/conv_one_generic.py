"""One generic-path conv forward + backward-data (shape from argv: N Cb Kb H W R S pad stride), for
compute-sanitizer / debugging."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05755_b200 as tpp  # noqa: E402
from paper_2104_05755_b200 import _lib  # noqa: E402

N, Cb, Kb, H, W, R, S, pad, st = (int(v) for v in sys.argv[1:10])
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
spec = tpp.ConvSpec(N, Cb, Kb, H, W, r=R, s=S, pad=pad, stride=st)
x = torch.rand(N * Cb * H * W * 64, generator=gen, device=dev).to(torch.bfloat16)
wv = (torch.randn(Kb * Cb * R * S * 64 * 64, generator=gen, device=dev) * 0.05).to(torch.bfloat16)
conv = tpp.Conv2d(spec, wv)
y = torch.empty(N * Kb * spec.p * spec.q * 64, dtype=torch.bfloat16, device=dev)
conv.forward(x, out=y)
torch.cuda.synchronize()
print("fwd", _lib.last_config(), flush=True)
dy = torch.randn_like(y)
dx = torch.empty_like(x)
conv.backward_data(dy, din=dx)
torch.cuda.synchronize()
print("bwd", _lib.last_config(), flush=True)
