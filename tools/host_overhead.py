import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_05755_b200 as tpp
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(0)
layer, x, out = bench.make_fc_set(torch, tpp, gen, dev, 16, 16, 64, 64, 16, 64, tpp.UnaryKind.RELU, 0.02, 0.02)
for _ in range(10): layer.forward(x, 16, 64, out=out)
torch.cuda.synchronize()
n = 2000
t = time.perf_counter()
for _ in range(n): layer.forward(x, 16, 64, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host us per forward call: {(t1 - t) / n * 1e6:.1f}; incl. drain {(time.perf_counter() - t) / n * 1e6:.1f}")
xh = torch.empty(x.numel(), dtype=torch.bfloat16, pin_memory=True)
oh = torch.empty(out.numel(), dtype=torch.bfloat16, pin_memory=True)
for name, fn in (("h2d", lambda: x.copy_(xh, non_blocking=True)), ("d2h", lambda: oh.copy_(out, non_blocking=True))):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 200
    print(f"{name}: {ms*1e3:.1f} us per 2 MiB = {2*2**20/ms/1e6:.1f} GB/s")
