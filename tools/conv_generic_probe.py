"""Timing of the generic (offset-BRGEMM composition) conv path on ResNet-50
shapes the fused kernels do not take: 3x3 stride 2 (56 -> 28), 1x1 stride 2
projection, 3x3 at 28x28 with C = K = 128 (two channel blocks), forward and
backward-data; CUDA graphs of K launches."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_05755_b200 as tpp  # noqa: E402

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
res = {}
for name, (N, Cb, Kb, H, W, R, S, pad, st) in {
        "3x3_s2_56to28_c64": (256, 1, 1, 56, 56, 3, 3, 1, 2),
        "1x1_s2_56to28_c64_k128": (256, 1, 2, 56, 56, 1, 1, 0, 2),
        "3x3_s1_28_c128": (256, 2, 2, 28, 28, 3, 3, 1, 1)}.items():
    spec = tpp.ConvSpec(N, Cb, Kb, H, W, r=R, s=S, pad=pad, stride=st)
    x = torch.rand(N * Cb * H * W * 64, generator=gen, device=dev).to(torch.bfloat16)
    wv = (torch.randn(Kb * Cb * R * S * 64 * 64, generator=gen, device=dev) * 0.05).to(torch.bfloat16)
    conv = tpp.Conv2d(spec, wv)
    y = torch.empty(N * Kb * spec.p * spec.q * 64, dtype=torch.bfloat16, device=dev)
    dy = torch.randn_like(y)
    dx = torch.empty_like(x)
    r = {"fused": spec.fused}
    for lab, fn in (("fwd", lambda: conv.forward(x, out=y)), ("bwd_data", lambda: conv.backward_data(dy, din=dx))):
        fn()
        g = bench.graph_of(torch, [fn] * 5)
        ms = statistics.median(bench.time_graph(torch, None, g, reps_min=5, min_seconds=0.3)) / 5
        r[lab] = {"us": round(ms * 1e3, 1), "TFLOP/s": round(spec.flops / ms / 1e9, 1)}
    res[name] = r
print(json.dumps(res))
