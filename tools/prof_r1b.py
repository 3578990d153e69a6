"""One launch each of the kernels added late in round 1 (for one ncu pass):
INT8 tcgen05 BRGEMM, DROPOUT (mask + scaled copy), cfg 3 FC1 with GELU."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2104_05755_b200 as tpp
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(0)
m = n = 4096; k, cnt = 1024, 8
a = torch.randint(-128, 128, (cnt * k * m,), generator=gen, device=dev, dtype=torch.int8)
b = torch.randint(-128, 128, (cnt * n * k,), generator=gen, device=dev, dtype=torch.int8)
c = tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.INT32), device=dev)
spec = tpp.GemmSpec(m, n, k, m, k, m, in_dtype=tpp.DType.INT8, out_dtype=tpp.DType.INT32)
tpp.brgemm(spec, tpp.BrgemmBatch.stride(a, b, k * m, n * k, cnt), c)
R, C = 8192, 4096
x = tpp.TensorView(tpp.TensorDesc(R, C, R, tpp.DType.BF16), torch.randn(R * C, generator=gen, device=dev).to(torch.bfloat16))
x.tertiary = {"prng": tpp.PrngState(1, C)}
y = tpp.alloc(tpp.TensorDesc(R, C, R, tpp.DType.BF16), device=dev)
tpp.apply_unary(tpp.UnaryKind.DROPOUT, x, y, dropout_p=0.1)
layer, xin, out = bench.make_fc_set(torch, tpp, gen, dev, 512, 16, 32, 64, 64, 64, tpp.UnaryKind.GELU, 1.0, 0.02, bias=False)
layer.forward(xin, 512, 32, out=out)
torch.cuda.synchronize()
