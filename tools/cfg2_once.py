"""One eager cfg2 FC launch (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_05755_b200 as tpp
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(0)
layer, x, out = bench.make_fc_set(torch, tpp, gen, dev, 16, 16, 64, 64, 16, 64, tpp.UnaryKind.RELU, 0.02, 0.02)
for _ in range(3):
    layer.forward(x, 16, 64, out=out)
torch.cuda.synchronize()
