"""DROPOUT / DROPOUT_INV timing on the bench shape (dense BF16 8192 x 4096
column-major views, 3 rotating operand sets > 2x L2), as bench.py's extra."""
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
R, C = 8192, 4096
res = {}
for dt, tdt in (("bf16", torch.bfloat16), ("fp32", torch.float32)):
    DT = tpp.DType.BF16 if dt == "bf16" else tpp.DType.FP32
    mk = lambda: tpp.TensorView(tpp.TensorDesc(R, C, R, DT), torch.randn(R * C, generator=gen, device=dev).to(tdt))  # noqa: E731
    sets = [(mk(), mk()) for _ in range(3)]
    for k in range(3):
        sets[k][0].tertiary = {"prng": tpp.PrngState(k, C)}
    g = bench.graph_of(torch, [(lambda k=k: tpp.apply_unary(tpp.UnaryKind.DROPOUT, sets[k][0], sets[k][1],
                                                           dropout_p=0.1)) for k in range(3)] * 2)
    ms = statistics.median(bench.time_graph(torch, None, g, reps_min=5, min_seconds=0.3)) / 6
    byts = 2 * R * C * (2 if dt == "bf16" else 4) + R * C // 8
    res[dt] = {"us": round(ms * 1e3, 2), "GB/s": round(byts / ms / 1e6, 1), "frac_hbm": round(byts / ms / 1e6 / 6552.6, 4)}
    del sets, g
print(json.dumps(res))
