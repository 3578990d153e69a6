"""Per-GEMM timing of the cfg-5 K=1024 shapes under the diagnostic modes of a
TPP_PHASE_STAMPS build (TPP_DBG_MODE: 1 = no epilogue math/stores, 2 = no
MMAs): is a tile bound by its mainloop or its epilogue?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05755_b200 as tpp  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
TOK = 8192


def bf(n, s=1.0):
    return (torch.randn(n, generator=g, device=dev) * s).to(torch.bfloat16)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps * 1e3, 2)


res = {"mode": os.environ.get("TPP_DBG_MODE", "0")}
L0 = tpp.FcLayer(64, 16, 64, 64, None, activation=tpp.UnaryKind.RELU, w_packed=bf(4096 * 1024, 0.02))
x0 = bf(TOK * 1024)
o0 = torch.empty(TOK * 4096, dtype=torch.bfloat16, device=dev)
m0 = torch.empty(TOK * 4096 // 8, dtype=torch.uint8, device=dev)
res["fwd0_relu_mask"] = timeit(lambda: L0.forward(x0, TOK // 64, 64, out=o0, relu_mask=m0))
res["fwd0_plain"] = timeit(lambda: L0.forward(x0, TOK // 64, 64, out=o0))
L1 = tpp.FcLayer(64, 64, 64, 64, None, activation=tpp.UnaryKind.RELU, w_packed=bf(4096 * 4096, 0.02))
x1 = bf(TOK * 4096)
res["fwd1_relu_mask"] = timeit(lambda: L1.forward(x1, TOK // 64, 64, out=o0, relu_mask=m0))
L3 = tpp.FcLayer(16, 64, 64, 64, None, w_packed=bf(1024 * 4096, 0.02))
d3 = bf(TOK * 1024)
res["dx3_relu_inv"] = timeit(lambda: L3.backward_data(d3, TOK // 64, 64, relu_mask_in=m0, out=o0))
print(json.dumps(res))
