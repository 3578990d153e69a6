"""e2e pipeline probe: which leg limits the per-step time (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_05755_b200 as tpp
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(0)
NB, CB, BN, BC, KB, BK = 16, 16, 64, 64, 16, 64
layer0, x0, _ = bench.make_fc_set(torch, tpp, gen, dev, NB, CB, BN, BC, KB, BK, tpp.UnaryKind.RELU, 0.02, 0.02)
n_in, n_out = NB * CB * BN * BC, NB * KB * BN * BK
x_host = torch.empty(n_in, dtype=torch.bfloat16, pin_memory=True)
out_host = [torch.empty(n_out, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
x_dev = [torch.empty(n_in, dtype=torch.bfloat16, device=dev) for _ in range(2)]
out_dev = [torch.empty(n_out, dtype=torch.bfloat16, device=dev) for _ in range(2)]
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
ev_in = [torch.cuda.Event() for _ in range(2)]
ev_comp = [torch.cuda.Event() for _ in range(2)]
ev_out = [torch.cuda.Event() for _ in range(2)]
def step(i, comp, h2d=True, d2h=True, kern=True):
    b = i % 2
    with torch.cuda.stream(s_in):
        if i >= 2: s_in.wait_event(ev_comp[b])
        if h2d: x_dev[b].copy_(x_host, non_blocking=True)
        ev_in[b].record(s_in)
    comp.wait_event(ev_in[b])
    if i >= 2: comp.wait_event(ev_out[b])
    if kern: layer0.forward(x_dev[b], NB, BN, out=out_dev[b], stream=comp)
    ev_comp[b].record(comp)
    with torch.cuda.stream(s_out):
        s_out.wait_event(ev_comp[b])
        if d2h: out_host[b].copy_(out_dev[b], non_blocking=True)
        ev_out[b].record(s_out)
K = 50
for name, kw in (("all", {}), ("no kernel", dict(kern=False)), ("no d2h", dict(d2h=False)), ("no h2d", dict(h2d=False)), ("kernel only", dict(h2d=False, d2h=False))):
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        cap = torch.cuda.current_stream()
        s_in.wait_stream(cap); s_out.wait_stream(cap)
        for i in range(K): step(i, cap, **kw)
        cap.wait_stream(s_in); cap.wait_stream(s_out)
    gr.replay(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
    print(f"{name:12s}: {e0.elapsed_time(e1) * 1e3 / K:7.1f} us per step")
