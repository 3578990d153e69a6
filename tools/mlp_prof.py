"""cfg 5 MLP training step: per-kernel breakdown (run under ncu --metrics gpu__time_duration.sum)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05755_b200 as tpp
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(0)
mlp = tpp.BlockedMLP([1024, 4096, 4096, 4096, 1024], 8192, bn=64, lr=0.01, device=dev, seed=7)
x = torch.randn(8192 * 1024, generator=gen, device=dev).to(torch.bfloat16)
tg = torch.randint(0, 1024, (8192,), generator=gen, device=dev, dtype=torch.int32)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(n):
    mlp.train_step(x, tg)
torch.cuda.synchronize()
print("ok")
