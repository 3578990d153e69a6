"""One cfg5 training step (eager), for ncu captures of every GEMM of the step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05755_b200 as tpp  # noqa: E402

dev = torch.device("cuda", 0)
mlp = tpp.BlockedMLP([1024, 4096, 4096, 4096, 1024], 8192, bn=64, lr=0.01, global_batch=8192, seed=7, device=dev)
g = torch.Generator(device=dev)
g.manual_seed(1)
x = torch.randn(8192 * 1024, generator=g, device=dev).to(torch.bfloat16)
tg = torch.randint(0, 1024, (8192,), generator=g, device=dev, dtype=torch.int32)
for _ in range(int(os.environ.get("STEPS", "2"))):
    mlp.train_step(x, tg)
torch.cuda.synchronize()
print("ok")
