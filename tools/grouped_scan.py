"""K11 per-stage cost: the cfg-2 composition with the batch length cut down
(count = 1 .. 16 entries per C block), one grouped launch, graph-timed."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_05755_b200 as tpp  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
Nb, Cb, bn, bc, Kb, bk = 16, 16, 64, 64, 16, 64
blk = bc * bk
x = torch.randn(Nb * Cb * blk, generator=g, device=dev).to(torch.bfloat16)
w = (torch.randn(Kb * Cb * blk, generator=g, device=dev) * 0.02).to(torch.bfloat16)
out = torch.empty(Nb * Kb * bn * bk, dtype=torch.float32, device=dev)
groups = [(nb, kb) for nb in range(Nb) for kb in range(Kb)]
res = {}
for vnni in (True, False):
    for cnt in (1, 2, 4, 8, 16):
        spec = tpp.GemmSpec(bk, bn, bc, bk, bc, bk, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32,
                            a_layout=tpp.ALayout.VNNI if vnni else tpp.ALayout.PLAIN)
        gb = tpp.GroupedBatch.stride(w, x, blk, blk, cnt, [kb * Cb * blk for _, kb in groups],
                                     [nb * Cb * blk for nb, _ in groups])
        co = [(nb * Kb + kb) * bn * bk for nb, kb in groups]
        gr = bench.graph_of(torch, [lambda: tpp.brgemm_grouped(spec, gb, out, co)] * 20)
        ms = statistics.median(bench.time_graph(torch, None, gr, reps_min=5, min_seconds=0.2)) / 20
        res[f"{'vnni' if vnni else 'plain'}_count{cnt}"] = round(ms * 1e3, 2)
print(json.dumps(res))
