import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_05755_b200 as tpp
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(0)
def run(nb, cb, kb, bn, block_n, label, bias=True, act=tpp.UnaryKind.RELU):
    layer, x, out = bench.make_fc_set(torch, tpp, gen, dev, nb, cb, bn, 64, kb, 64, act, 0.02, 0.02, bias=bias)
    layer.block_n = block_n
    g = bench.graph_of(torch, [lambda: layer.forward(x, nb, bn, out=out)] * 20)
    ms = statistics.median(bench.time_graph(torch, None, g, reps_min=10, min_seconds=0.3)) / 20
    fl = 2 * nb * bn * cb * 64 * kb * 64
    print(f"KPS={os.environ.get('TPP_KPS','auto')} {label:34s} bn_tile={block_n:4d}: {ms*1e3:8.2f} us  {fl/ms/1e9:7.1f} TFLOP/s")
run(16, 16, 16, 64, 64, "cfg2")
run(16, 16, 16, 64, 64, "cfg2 no bias", bias=False)
run(16, 16, 16, 64, 64, "cfg2 no bias no act", bias=False, act=None)
run(16, 1, 16, 64, 64, "K=64 (1 k-block)")
run(16, 4, 16, 64, 64, "K=256")
run(512, 64, 16, 32, 256, "cfg3 FC2 (K=4096,N=1024)", bias=False, act=None)
run(512, 16, 64, 32, 256, "cfg3 FC1 (K=1024,N=4096)", bias=False, act=tpp.UnaryKind.GELU)
run(512, 16, 64, 32, 128, "cfg3 FC1 BN=128", bias=False, act=tpp.UnaryKind.GELU)
