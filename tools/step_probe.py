"""cfg5 step timing probe: graph-replayed vs eager vs per-launch breakdown
(bench.py's pieces), one JSON line; run with and without TPP_NO_PDL."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_05755_b200 as tpp  # noqa: E402

K = int(os.environ.get("K", "20"))
dev = torch.device("cuda", 0)
mlp = tpp.BlockedMLP(bench.DIMS, 8192, bn=64, lr=0.01, global_batch=8192, seed=7, device=dev,
                     defer_join=os.environ.get("DEFER", "1") == "1")
gen = torch.Generator(device=dev)
gen.manual_seed(1)
x = torch.randn(8192 * 1024, generator=gen, device=dev).to(torch.bfloat16)
tg = torch.randint(0, 1024, (8192,), generator=gen, device=dev, dtype=torch.int32)
step = lambda: mlp.train_step(x, tg)  # noqa: E731
for _ in range(5):
    step()
mlp.sync_updates()
torch.cuda.synchronize()
out = {"pdl": os.environ.get("TPP_NO_PDL") is None}
g = bench.graph_of(torch, [step] * K + [mlp.sync_updates])
out["graph_ms"] = statistics.median(bench.time_graph(torch, None, g, reps_min=10, min_seconds=1.0)) / K
out["eager_ms"] = statistics.median(bench.time_eager(torch, None, step, K, reps=10, tail=mlp.sync_updates)) / K
out["graph_ms_2"] = statistics.median(bench.time_graph(torch, None, g, reps_min=10, min_seconds=1.0)) / K
out["eager_ms_2"] = statistics.median(bench.time_eager(torch, None, step, K, reps=10, tail=mlp.sync_updates)) / K
bd = bench.step_breakdown(torch, mlp, x, tg, K)
out["breakdown_sum_ms"] = sum(bd.values())
out["breakdown"] = {k: round(v, 4) for k, v in bd.items()}
out["graph_ms_again"] = statistics.median(bench.time_graph(torch, None, g, reps_min=10, min_seconds=1.0)) / K
print(json.dumps(out))
