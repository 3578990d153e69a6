import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_05755_b200 as tpp
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(0)
def run(nb, cb, kb, bn, block_n, label):
    layer, x, out = bench.make_fc_set(torch, tpp, gen, dev, nb, cb, bn, 64, kb, 64, tpp.UnaryKind.RELU, 0.02, 0.02)
    layer.block_n = block_n
    g = bench.graph_of(torch, [lambda: layer.forward(x, nb, bn, out=out)] * 20)
    ms = statistics.median(bench.time_graph(torch, None, g, reps_min=10, min_seconds=0.3)) / 20
    fl = 2 * nb * bn * cb * 64 * kb * 64
    print(f"{label:40s} block_n={block_n:4d}: {ms*1e3:8.2f} us  {fl/ms/1e9:7.1f} TFLOP/s (warm L2)")
for bnt in (64, 128, 256):
    run(16, 16, 16, 64, bnt, "cfg2 1024^3")
for kbl in (8, 32, 64):
    run(16, kbl, 16, 64, 64, f"N=1024 K={kbl*64} M=1024")
run(32, 16, 32, 64, 64, "N=2048 C=1024 K=2048")
run(148*2, 16, 8, 64, 256, "N=18944 C=1024 K=512 (148x2 tiles)")
