"""Run one hot-path op a few times (no graphs) for ncu / compute-sanitizer.

    python tools/prof.py cfg2|fc1|fc2|conv|convbwd|ln|brgemm1 [--iters N]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_05755_b200 as tpp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("op")
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    if a.op == "cfg2":
        layer, x, out = bench.make_fc_set(torch, tpp, gen, dev, 16, 16, 64, 64, 16, 64,
                                          tpp.UnaryKind.RELU, 0.02, 0.02)
        fn = lambda: layer.forward(x, 16, 64, out=out)  # noqa: E731
    elif a.op in ("fc1", "fc2"):
        nb, bn = 512, 32
        cin, cout = (16, 64) if a.op == "fc1" else (64, 16)
        act = tpp.UnaryKind.GELU if a.op == "fc1" else None
        layer, x, out = bench.make_fc_set(torch, tpp, gen, dev, nb, cin, bn, 64, cout, 64, act, 1.0, 0.02,
                                          bias=False)
        res = torch.randn(out.numel(), generator=gen, device=dev).to(torch.bfloat16) if a.op == "fc2" else None
        fn = lambda: layer.forward(x, nb, bn, out=out, residual=res)  # noqa: E731
    elif a.op in ("conv", "convbwd"):
        spec = tpp.ConvSpec(256, 1, 1, 56, 56)
        x = torch.rand(256 * 56 * 56 * 64, generator=gen, device=dev).to(torch.bfloat16)
        w = (torch.randn(9 * 64 * 64, generator=gen, device=dev) * 0.06).to(torch.bfloat16)
        conv = tpp.Conv2d(spec, w)
        y = torch.empty_like(x)
        fn = (lambda: conv.forward(x, out=y)) if a.op == "conv" else (lambda: conv.backward_data(x, din=y))
    elif a.op == "convdw":
        spec = tpp.ConvSpec(256, 1, 1, 56, 56)
        x = torch.rand(256 * 56 * 56 * 64, generator=gen, device=dev).to(torch.bfloat16)
        dy = torch.randn(256 * 56 * 56 * 64, generator=gen, device=dev).to(torch.bfloat16)
        wv = (torch.randn(9 * 64 * 64, generator=gen, device=dev) * 0.1).to(torch.bfloat16)
        conv = tpp.Conv2d(spec, wv)
        fn = lambda: conv.backward_weights(x, dy)  # noqa: E731
    elif a.op == "ln":
        x = torch.randn(16384 * 1024, generator=gen, device=dev).to(torch.bfloat16)
        o = torch.empty_like(x)
        fn = lambda: tpp.layernorm_blocked(x, 512, 16, 32, 64, 1e-5, out=o)  # noqa: E731
    elif a.op == "brgemm1":
        m = n = k = 64
        A = torch.rand(m * k * 16, generator=gen, device=dev)
        B = torch.rand(k * n * 16, generator=gen, device=dev)
        c = tpp.TensorView(tpp.TensorDesc(m, n, m, tpp.DType.FP32), torch.rand(m * n, device=dev))
        sp = tpp.GemmSpec(m, n, k, m, k, m, beta=1.0)
        bt = tpp.BrgemmBatch.stride(A, B, m * k, k * n, 16)
        fn = lambda: tpp.brgemm(sp, bt, c)  # noqa: E731
    else:
        raise SystemExit(f"unknown op {a.op}")
    for _ in range(a.iters):
        fn()
    torch.cuda.synchronize()
    print("ok", a.op)


if __name__ == "__main__":
    main()
