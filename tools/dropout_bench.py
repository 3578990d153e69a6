"""Time DROPOUT / DROPOUT_INV / PRNG fill on the GPU (CUDA events, L2 flushed
by rotating input sets larger than L2) and print achieved HBM GB/s."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2104_05755_b200 as tpp  # noqa: E402


def timeit(fn, iters=30):
    """Launches captured in a CUDA graph so host (ctypes) overhead is out of
    the device timing."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(3):
            fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(iters):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / iters)
    return best


def main():
    for rows, cols, dt in ((4096, 4096, tpp.DType.FP32), (4096, 4096, tpp.DType.BF16), (1024, 16384, tpp.DType.BF16)):
        esz = 4 if dt is tpp.DType.FP32 else 2
        sets = []
        for s in range(3):
            x = tpp.from_array(np.random.default_rng(s).standard_normal((rows, cols)).astype(np.float32), dt)
            x.tertiary = {"prng": tpp.PrngState(s, cols)}
            out = tpp.alloc(tpp.TensorDesc(rows, cols, rows, dt))
            sets.append((x, out))

        def drop(i):
            x, out = sets[i % 3]
            tpp.apply_unary(tpp.UnaryKind.DROPOUT, x, out, dropout_p=0.1)

        us = timeit(drop)
        byts = rows * cols * esz * 2 + rows * cols / 8
        print(f"DROPOUT {dt.name} {rows}x{cols}: {us:.1f} us  {byts / us / 1e3:.0f} GB/s", flush=True)
        for x, out in sets:
            x.secondary = out.secondary

        def inv(i):
            x, out = sets[i % 3]
            tpp.apply_unary(tpp.UnaryKind.DROPOUT_INV, x, out, dropout_p=0.1)

        us = timeit(inv)
        print(f"DROPOUT_INV {dt.name} {rows}x{cols}: {us:.1f} us  {byts / us / 1e3:.0f} GB/s", flush=True)

        def relu_inv(i):
            x, out = sets[i % 3]
            tpp.apply_unary(tpp.UnaryKind.RELU_INV, x, out)

        us = timeit(relu_inv)
        print(f"  (RELU_INV same shape: {us:.1f} us  {byts / us / 1e3:.0f} GB/s)", flush=True)

        def copy(i):
            x, out = sets[i % 3]
            out.primary.copy_(x.primary)

        us = timeit(copy)
        print(f"  (torch copy same shape: {us:.1f} us  {(byts - rows * cols / 8) / us / 1e3:.0f} GB/s)", flush=True)
    outs = [tpp.alloc(tpp.TensorDesc(4096, 4096, 4096, tpp.DType.FP32)) for _ in range(3)]
    src = tpp.alloc(tpp.TensorDesc(1, 1, 1, tpp.DType.FP32))
    src.tertiary = {"prng": tpp.PrngState(1, 4096)}
    us = timeit(lambda i: tpp.apply_unary(tpp.UnaryKind.PRNG, src, outs[i % 3]))
    print(f"PRNG fill FP32 4096x4096: {us:.1f} us  {4096 * 4096 * 4 / us / 1e3:.0f} GB/s", flush=True)


def ncu_mode():
    """One eager launch of each kernel on 4096 x 4096 BF16 (for ncu)."""
    rows = cols = 4096
    x = tpp.from_array(np.random.default_rng(0).standard_normal((rows, cols)).astype(np.float32), tpp.DType.BF16)
    x.tertiary = {"prng": tpp.PrngState(0, cols)}
    out = tpp.alloc(tpp.TensorDesc(rows, cols, rows, tpp.DType.BF16))
    tpp.apply_unary(tpp.UnaryKind.DROPOUT, x, out, dropout_p=0.1)
    x.secondary = out.secondary
    tpp.apply_unary(tpp.UnaryKind.DROPOUT_INV, x, out, dropout_p=0.1)
    torch.cuda.synchronize()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "ncu":
    ncu_mode()
    sys.exit(0)


if __name__ == "__main__":
    main()
