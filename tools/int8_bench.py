"""INT8 BRGEMM on tcgen05 kind::i8: TOPS for a few STRIDE shapes (CUDA-graph
timed, so ctypes overhead is out of the device timing)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2104_05755_b200 as tpp  # noqa: E402
from dropout_bench import timeit  # noqa: E402


def run(m, n, k, count, engine=tpp.Engine.AUTO, iters=20):
    rng = np.random.default_rng(0)
    a = torch.from_numpy(rng.integers(-128, 128, count * k * m, dtype=np.int8)).cuda()
    b = torch.from_numpy(rng.integers(-128, 128, count * n * k, dtype=np.int8)).cuda()
    cs = [tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.INT32)) for _ in range(2)]
    spec = tpp.GemmSpec(m, n, k, m, k, m, in_dtype=tpp.DType.INT8, out_dtype=tpp.DType.INT32, engine=engine)
    batch = tpp.BrgemmBatch.stride(a, b, k * m, n * k, count)
    us = timeit(lambda i: tpp.brgemm(spec, batch, cs[i % 2]), iters)
    tops = 2.0 * m * n * k * count / us / 1e6
    print(f"INT8 {engine.name:7s} M={m} N={n} K={k} x{count}: {us:9.1f} us  {tops:7.1f} TOPS", flush=True)


if __name__ == "__main__":
    run(64, 64, 64, 16)
    run(1024, 1024, 1024, 4)
    run(4096, 4096, 4096, 1)
    run(8192, 8192, 2048, 2)
    run(4096, 4096, 1024, 8)
    run(1024, 1024, 1024, 1, tpp.Engine.ORDERED, iters=3)
