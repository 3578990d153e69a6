"""cfg3 FC1 (16384 x 1024 -> 4096, GELU) and FC2 (+ residual) timing, bench.py's
method; run with and without TPP_NO_TMA_STORE=1 (epilogue stores straight from
registers instead of smem staging + TMA stores)."""
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
nb, bn, h, f = 512, 32, 16, 64
x = torch.randn(nb * h * bn * 64, generator=gen, device=dev).to(torch.bfloat16)
w1 = (torch.randn(f, h, 64, 64, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
w2 = (torch.randn(h, f, 64, 64, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
fc1 = tpp.FcLayer(f, h, 64, 64, bench._vnni_from_logical(w1).reshape(-1), activation=tpp.UnaryKind.GELU)
fc2 = tpp.FcLayer(h, f, 64, 64, bench._vnni_from_logical(w2).reshape(-1))
fc1n = tpp.FcLayer(f, h, 64, 64, bench._vnni_from_logical(w1).reshape(-1))            # no activation
fc1r = tpp.FcLayer(f, h, 64, 64, bench._vnni_from_logical(w1).reshape(-1), activation=tpp.UnaryKind.RELU)
mid = torch.empty(nb * f * bn * 64, dtype=torch.bfloat16, device=dev)
o2 = torch.empty(nb * h * bn * 64, dtype=torch.bfloat16, device=dev)
fl = 2 * 16384 * 1024 * 4096
mode = "off" if os.environ.get("TPP_NO_TMA_STORE") else "on"
for name, fn in (("fc1_gelu", lambda: fc1.forward(x, nb, bn, out=mid)),
                 ("fc1_none", lambda: fc1n.forward(x, nb, bn, out=mid)),
                 ("fc1_relu", lambda: fc1r.forward(x, nb, bn, out=mid)),
                 ("fc2_residual", lambda: fc2.forward(mid, nb, bn, out=o2, residual=x))):
    g = bench.graph_of(torch, [fn] * 10)
    ms = statistics.median(bench.time_graph(torch, None, g, reps_min=10, min_seconds=0.5)) / 10
    print(f"{name:13s} tma_store={mode:3s} {ms * 1e3:8.2f} us {fl / ms / 1e9:7.1f} TFLOP/s  {_lib.last_config()}")
