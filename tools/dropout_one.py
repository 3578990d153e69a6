"""One DROPOUT TPP call on the bench shape (BF16 8192 x 4096), a few times, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05755_b200 as tpp  # noqa: E402

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
R, C = 8192, 4096
dt = tpp.DType.FP32 if os.environ.get("FP32") else tpp.DType.BF16
tdt = torch.float32 if os.environ.get("FP32") else torch.bfloat16
x = tpp.TensorView(tpp.TensorDesc(R, C, R, dt), torch.randn(R * C, generator=gen, device=dev).to(tdt))
y = tpp.TensorView(tpp.TensorDesc(R, C, R, dt), torch.empty(R * C, device=dev).to(tdt))
x.tertiary = {"prng": tpp.PrngState(1, C)}
for _ in range(4):
    tpp.apply_unary(tpp.UnaryKind.DROPOUT, x, y, dropout_p=0.1)
torch.cuda.synchronize()
print("ok")
