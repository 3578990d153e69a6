"""Host (Python + ctypes) cost of the public API calls, GPU drained separately:
the cfg-5 BlockedMLP.train_step (12 launches) and one FcLayer.forward (cfg 2)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_05755_b200 as tpp  # noqa: E402

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
mlp = tpp.BlockedMLP(bench.DIMS, 8192, bn=64, lr=0.01, global_batch=8192, seed=7, device=dev)
x = torch.randn(8192 * 1024, generator=gen, device=dev).to(torch.bfloat16)
tg = torch.randint(0, 1024, (8192,), generator=gen, device=dev, dtype=torch.int32)
for _ in range(5):
    mlp.train_step(x, tg)
torch.cuda.synchronize()
n = 50
t0 = time.perf_counter()
for _ in range(n):
    mlp.train_step(x, tg)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"cfg5 train_step: host {((t1 - t0) / n) * 1e6:.1f} us per step (12 launches), "
      f"wall incl. drain {((t2 - t0) / n) * 1e6:.1f} us per step -> the GPU stays ahead of the host")
wl = (torch.randn(16, 16, 64, 64, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
layer = tpp.FcLayer(16, 16, 64, 64, bench._vnni_from_logical(wl).reshape(-1),
                    bias=torch.zeros(1024, device=dev, dtype=torch.bfloat16), activation=tpp.UnaryKind.RELU)
xi = torch.randn(16 * 16 * 64 * 64, generator=gen, device=dev).to(torch.bfloat16)
o = torch.empty_like(xi)
for _ in range(10):
    layer.forward(xi, 16, 64, out=o)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    layer.forward(xi, 16, 64, out=o)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"cfg2 FcLayer.forward: host {((t1 - t0) / n) * 1e6:.1f} us per call (validation, ctypes, 3 tensor-map "
      f"encodes, launch), wall incl. drain {((t2 - t0) / n) * 1e6:.1f} us per call; the kernel alone is ~6.5 us")
