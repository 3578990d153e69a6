"""cfg 2 fixed-latency floor: the same launch (128 tiles of 128 x 64 on 148
SMs, bias + ReLU epilogue, BF16 out) with K = 1024 (the real layer), 512,
256, 128 and 64 -- CUDA graph of 20 launches on rotating sets, per-launch
time.  The K -> 0 intercept is the cost no mainloop speed-up can remove."""
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
for cb in (16, 8, 4, 2, 1):
    sets = []
    for _ in range(20):
        x = (torch.randn(16 * cb * 64 * 64, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
        wl = (torch.randn(16, cb, 64, 64, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
        b = (torch.randn(1024, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
        L = tpp.FcLayer(16, cb, 64, 64, bench._vnni_from_logical(wl).reshape(-1), bias=b, activation=tpp.UnaryKind.RELU)
        sets.append((L, x, torch.empty(16 * 16 * 64 * 64, dtype=torch.bfloat16, device=dev)))
    g = bench.graph_of(torch, [(lambda s=s: s[0].forward(s[1], 16, 64, out=s[2])) for s in sets])
    ms = statistics.median(bench.time_graph(torch, None, g, reps_min=10, min_seconds=0.5)) / 20
    fl = 2 * 1024 * 1024 * 64 * cb
    res[f"K={64 * cb}"] = {"us": round(ms * 1e3, 3), "TFLOP/s": round(fl / ms / 1e9, 1)}
    del sets, g
print(json.dumps(res))
