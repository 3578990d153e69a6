"""One cfg5 forward GEMM (8192 tokens x 4096 -> 4096, ReLU + bitmask: the
CTA-pair kernel brgemm_tc_kernel<256,3,2,0,2,1>) launched a few times — the
target of the ncu --set full capture behind bench.py's roofline.traffic."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05755_b200 as tpp  # noqa: E402
from paper_2104_05755_b200 import _lib  # noqa: E402
from paper_2104_05755_b200 import training as T  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
D, TOK = 4096, 8192
C = int(os.environ.get("K_IN", "4096"))  # reduce width: 1024 = the cfg5 fwd0 shape
w = T.pack_logical_weight((torch.randn(D, C, generator=g, device=dev) * 0.02).to(torch.bfloat16))
layer = tpp.FcLayer(D // 64, C // 64, 64, 64, None, activation=tpp.UnaryKind.RELU, w_packed=w)
x = torch.randn(TOK * C, generator=g, device=dev).to(torch.bfloat16)
out = torch.empty(TOK * D, dtype=torch.bfloat16, device=dev)
mask = torch.empty(TOK * D // 8, dtype=torch.uint8, device=dev)
for _ in range(int(os.environ.get("REPS", "5"))):
    layer.forward(x, TOK // 64, 64, out=out, relu_mask=mask)
torch.cuda.synchronize()
print(_lib.last_config())
