"""H2D / D2H concurrency check for the e2e pipeline (diagnostics)."""
import torch
dev = torch.device("cuda", 0)
n = 1 << 20  # bf16 elements = 2 MiB
xh = [torch.empty(n, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
oh = [torch.empty(n, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
xd = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(2)]
od = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(mode, K=50):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
    for i in range(K):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1): xd[i % 2].copy_(xh[i % 2], non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2): oh[i % 2].copy_(od[i % 2], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    e1.record(); torch.cuda.synchronize()
    print(f"{mode}: {e0.elapsed_time(e1) * 1e3 / K:.1f} us per step")
for m in ("h2d", "d2h", "both", "both"):
    run(m)
