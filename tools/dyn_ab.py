"""Dynamic vs static tile scheduling on single cfg-5 GEMMs (graphs of K
back-to-back launches, replayed interleaved R rounds).  One JSON line of
median microseconds per launch."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_05755_b200 as tpp  # noqa: E402
from paper_2104_05755_b200 import _lib  # noqa: E402

K = int(os.environ.get("K", "10"))
R = int(os.environ.get("R", "5"))
dev = torch.device("cuda", 0)
lib = _lib.load()
T = 8192
shapes = {"fwd 4096->4096": (4096, 4096), "fwd 1024->4096": (1024, 4096), "fwd 4096->1024": (4096, 1024)}
keep, graphs, cfgs = [], {}, {}
for name, (ci, co) in shapes.items():
    w = (torch.randn(co * ci, device=dev) * 0.02).to(torch.bfloat16)
    layer = tpp.FcLayer(co // 64, ci // 64, 64, 64, None, activation=tpp.UnaryKind.RELU, w_packed=w)
    x = torch.randn(T * ci, device=dev).to(torch.bfloat16)
    out = torch.empty(T * co, device=dev, dtype=torch.bfloat16)
    mask = torch.empty(T * co // 8, device=dev, dtype=torch.uint8)
    keep += [w, layer, x, out, mask]
    for dyn in (1, 2):
        lib.tpp_set_tile_scheduling(dyn)
        fn = lambda L=layer, x=x, o=out, m=mask: L.forward(x, T // 64, 64, out=o, relu_mask=m)  # noqa: E731
        fn()
        torch.cuda.synchronize()
        cfgs[f"{name} {'dyn' if dyn == 1 else 'static'}"] = _lib.last_config()
        graphs[f"{name} {'dyn' if dyn == 1 else 'static'}"] = bench.graph_of(torch, [fn] * K)
# backward shapes of the step: dX (RELU_INV) and dW + split-SGD
for name, (ci, co) in {"dX 4096<-4096": (4096, 4096), "dX 4096<-1024": (4096, 1024)}.items():
    w = (torch.randn(co * ci, device=dev) * 0.02).to(torch.bfloat16)
    layer = tpp.FcLayer(co // 64, ci // 64, 64, 64, None, w_packed=w)
    dy = torch.randn(T * co, device=dev).to(torch.bfloat16)
    dx = torch.empty(T * ci, device=dev, dtype=torch.bfloat16)
    mask = torch.randint(0, 255, (T * ci // 8,), device=dev, dtype=torch.uint8)
    keep += [w, layer, dy, dx, mask]
    for dyn in (1, 2):
        lib.tpp_set_tile_scheduling(dyn)
        fn = lambda L=layer, dy=dy, dx=dx, m=mask: L.backward_data(dy, T // 64, 64, relu_mask_in=m, out=dx)  # noqa: E731
        fn()
        torch.cuda.synchronize()
        cfgs[f"{name} {'dyn' if dyn == 1 else 'static'}"] = _lib.last_config()
        graphs[f"{name} {'dyn' if dyn == 1 else 'static'}"] = bench.graph_of(torch, [fn] * K)
for name, (ci, co) in {"dW+SGD 4096x4096": (4096, 4096), "dW+SGD 1024x4096": (4096, 1024)}.items():
    w = (torch.randn(co * ci, device=dev) * 0.02).to(torch.bfloat16)
    lo = torch.zeros(co * ci, device=dev, dtype=torch.int16)
    layer = tpp.FcLayer(co // 64, ci // 64, 64, 64, None, w_packed=w)
    dy = torch.randn(T * co, device=dev).to(torch.bfloat16)
    x = torch.randn(T * ci, device=dev).to(torch.bfloat16)
    keep += [w, lo, layer, dy, x]
    for dyn in (1, 2):
        lib.tpp_set_tile_scheduling(dyn)
        fn = lambda L=layer, dy=dy, x=x, lo=lo: L.backward_weights_sgd(dy, x, T // 64, 64, lo, 1e-9)  # noqa: E731
        fn()
        torch.cuda.synchronize()
        cfgs[f"{name} {'dyn' if dyn == 1 else 'static'}"] = _lib.last_config()
        graphs[f"{name} {'dyn' if dyn == 1 else 'static'}"] = bench.graph_of(torch, [fn] * K)
lib.tpp_set_tile_scheduling(0)
res = {k: [] for k in graphs}
for _ in range(R):
    for k, g in graphs.items():
        res[k] += bench.time_graph(torch, None, g, reps_min=5, min_seconds=0.2)
out = {k: round(1000 * statistics.median(v) / K, 2) for k, v in res.items()}
out["configs"] = cfgs
print(json.dumps(out))
