"""Epilogue phase clocks (clock64, CTA 0, warp 4, tile 0) of the cfg2 FC
launch: acc ready -> TMEM loaded -> math done -> staged -> store issued ->
store read done -> exit."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_05755_b200 as tpp
from paper_2104_05755_b200 import _lib
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(0)
lib = _lib.load()
buf = torch.zeros(200, dtype=torch.int64, device=dev)
layer, x, out = bench.make_fc_set(torch, tpp, gen, dev, 16, 16, 64, 64, 16, 64, tpp.UnaryKind.RELU, 0.02, 0.02)
for it in range(3):
    buf.zero_()
    lib.tpp_debug_phase_timestamps(buf.data_ptr())
    g = bench.graph_of(torch, [lambda: layer.forward(x, 16, 64, out=out)] * 20)
    lib.tpp_debug_phase_timestamps(None)
    g.replay(); torch.cuda.synchronize()
    t = buf.cpu().tolist()
    base = t[189]
    names = ["tmem ld done", "math done", "staged", "store issued"]
    parts = [f"{n}={t[150 + i] - base}" for i, n in enumerate(names)]
    print("cycles after acc ready: ld issued", t[188] - base, " ".join(parts), f"pre-final-wait={t[190] - base} read-done={t[191] - base} exit={t[192] - base}")
