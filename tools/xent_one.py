"""The cfg5 softmax-CE gradient kernel alone (8192 tokens x 1024 classes,
blocked FP32 logits -> BF16 dlogits + per-token loss), a few launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05755_b200 as tpp  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
T_, C_ = 8192, 1024
logits = torch.randn(T_ * C_, generator=g, device=dev) * 3
tg = torch.randint(0, C_, (T_,), generator=g, device=dev, dtype=torch.int32)
d = torch.empty(T_ * C_, dtype=torch.bfloat16, device=dev)
loss = torch.empty(T_, dtype=torch.float32, device=dev)
reps = int(os.environ.get("REPS", "5"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(reps + 1):
    if i == 1:
        e0.record()
    tpp.softmax_xent_blocked(logits, tg, T_ // 64, C_ // 64, 64, 64, 1.0 / T_, dlogits=d, loss=loss)
e1.record()
torch.cuda.synchronize()
print(f"xent {e0.elapsed_time(e1) / reps * 1e3:.1f} us per launch")
