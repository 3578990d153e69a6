"""cfg5 step A/B in one process: {default (dynamic for the overlapped GEMMs), static} tile scheduling x
{overlapped, serial} backward.  Each variant is captured once as a CUDA graph
of K steps; the graphs are replayed interleaved (R rounds) so clock drift hits
every variant alike.  One JSON line: median ms per step per variant."""
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
gen = torch.Generator(device=dev)
gen.manual_seed(1)
x = torch.randn(8192 * 1024, generator=gen, device=dev).to(torch.bfloat16)
tg = torch.randint(0, 1024, (8192,), generator=gen, device=dev, dtype=torch.int32)
graphs = {}
keep = []  # the graphs read the models' buffers
for mode in ("deferred", "overlap", "serial"):
    mlp = tpp.BlockedMLP(bench.DIMS, 8192, bn=64, lr=0.01, global_batch=8192, seed=7, device=dev,
                         overlap=mode != "serial", defer_join=mode == "deferred")
    keep.append(mlp)
    for dyn in (0, 2):   # 0: the default (overlapped GEMMs dynamic), 2: every GEMM static
        if mode == "deferred" and dyn == 2:
            continue
        lib.tpp_set_tile_scheduling(dyn)
        step = lambda m=mlp: m.train_step(x, tg)  # noqa: E731
        for _ in range(3):
            step()
        mlp.sync_updates()
        torch.cuda.synchronize()
        graphs[f"{'default' if dyn == 0 else 'static'}+{mode}"] = bench.graph_of(torch, [step] * K + [mlp.sync_updates])
lib.tpp_set_tile_scheduling(0)
res = {k: [] for k in graphs}
for _ in range(R):
    for k, g in graphs.items():
        res[k] += bench.time_graph(torch, None, g, reps_min=3, min_seconds=0.3)
out = {k: round(statistics.median(v) / K, 5) for k, v in res.items()}
out["K"], out["R"] = K, R
print(json.dumps(out))
