"""The cfg-2 composition as ONE grouped tcgen05 BRGEMM launch (a few times),
for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05755_b200 as tpp  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
Nb, Cb, bn, bc, Kb, bk = 16, 16, 64, 64, 16, 64
blk = bc * bk
x = torch.randn(Nb * Cb * blk, generator=g, device=dev).to(torch.bfloat16)
w = (torch.randn(Kb * Cb * blk, generator=g, device=dev) * 0.02).to(torch.bfloat16)
out = torch.empty(Nb * Kb * bn * bk, dtype=torch.float32, device=dev)
spec = tpp.GemmSpec(bk, bn, bc, bk, bc, bk, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32, a_layout=tpp.ALayout.VNNI)
groups = [(nb, kb) for nb in range(Nb) for kb in range(Kb)]
gb = tpp.GroupedBatch.stride(w, x, blk, blk, Cb, [kb * Cb * blk for _, kb in groups], [nb * Cb * blk for nb, _ in groups])
for _ in range(5):
    tpp.brgemm_grouped(spec, gb, out, [(nb * Kb + kb) * bn * bk for nb, kb in groups])
torch.cuda.synchronize()
print("ok")
