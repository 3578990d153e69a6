"""Per-GEMM timing of the cfg5 small / tail-heavy shapes (stream-K on/off via
TPP_NO_STREAMK): fwd3 (8192x4096 -> 1024, FP32 out), dW 4096x4096 over 8192
tokens (+SGD), dW 1024x4096, fwd0 (8192x1024 -> 4096)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05755_b200 as tpp  # noqa: E402
from paper_2104_05755_b200 import _lib  # noqa: E402

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
    return e0.elapsed_time(e1) / reps * 1e3


res = {}
for name, (o, i) in {"fwd3": (1024, 4096), "fwd0": (4096, 1024), "fwd1": (4096, 4096)}.items():
    L = tpp.FcLayer(o // 64, i // 64, 64, 64, None, w_packed=bf(o * i, 0.02))
    x = bf(TOK * i)
    out = torch.empty(TOK * o, dtype=torch.float32 if name == "fwd3" else torch.bfloat16, device=dev)
    res[name] = timeit(lambda: L.forward(x, TOK // 64, 64, out=out))
    res[name + "_cfg"] = _lib.last_config()
for name, (o, i) in {"dw2": (4096, 4096), "dw3": (1024, 4096), "dw0": (4096, 1024)}.items():
    w = bf(o * i, 0.02)
    L = tpp.FcLayer(o // 64, i // 64, 64, 64, None, w_packed=w)
    lo = torch.zeros(o * i, dtype=torch.int16, device=dev)
    dy, x = bf(TOK * o, 1e-3), bf(TOK * i)
    res[name] = timeit(lambda: L.backward_weights_sgd(dy, x, TOK // 64, 64, lo, 1e-6))
    res[name + "_cfg"] = _lib.last_config()
res["streamk"] = os.environ.get("TPP_NO_STREAMK") is None
print(json.dumps(res))
