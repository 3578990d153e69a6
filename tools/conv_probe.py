"""cfg 4 conv timing (fwd / bwd-data / bwd-weights), bench.py's method."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_05755_b200 as tpp  # noqa: E402
from paper_2104_05755_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
spec = tpp.ConvSpec(256, 1, 1, 56, 56)
xin = torch.rand(256 * 56 * 56 * 64, generator=gen, device=dev).to(torch.bfloat16)
wl = (torch.randn(1, 1, 3, 3, 64, 64, generator=gen, device=dev) * (2 / 576) ** 0.5).to(torch.bfloat16)
wv = wl.reshape(1, 1, 3, 3, 64, 32, 2).permute(0, 1, 2, 3, 5, 4, 6).contiguous().reshape(-1)
conv = tpp.Conv2d(spec, wv)
yo = torch.empty_like(xin)
dO = torch.randn(256 * 56 * 56 * 64, generator=gen, device=dev).to(torch.bfloat16)
dI = torch.empty_like(xin)
res = {}
for name, fn in (("fwd", lambda: conv.forward(xin, out=yo)), ("bwd_data", lambda: conv.backward_data(dO, din=dI))):
    g = bench.graph_of(torch, [fn] * 5)
    ms = statistics.median(bench.time_graph(torch, None, g, reps_min=5, min_seconds=0.3)) / 5
    tf = spec.flops / ms / 1e9
    res[name] = {"us": round(ms * 1e3, 2), "TFLOP/s": round(tf, 1), "frac": round(tf / 1681.7, 4), "cfg": _lib.last_config()}
print(json.dumps(res))
