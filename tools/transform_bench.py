"""Standalone layout TPPs (TRANSPOSE / VNNI / VNNI_TO_VNNIT) and eltwise: GB/s vs HBM."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_05755_b200 as tpp
from paper_2104_05755_b200.ops import TransformKind, TransformSpec, transform
dev = torch.device("cuda", 0)
R = C = 8192  # 128 MiB per BF16 operand: every launch streams from HBM (> L2)
hbm = 6454.3
def timeit(fn, nbytes, label):
    g = bench.graph_of(torch, [fn] * 10)
    ms = statistics.median(bench.time_graph(torch, None, g, reps_min=5, min_seconds=0.3)) / 10
    print(f"{label:40s} {ms*1e3:8.1f} us  {nbytes/ms/1e6:8.1f} GB/s  {nbytes/ms/1e6/hbm*100:5.1f} % HBM")
for dt, tdt in ((tpp.DType.BF16, torch.bfloat16), (tpp.DType.FP32, torch.float32)):
    x = tpp.TensorView(tpp.TensorDesc(R, C, R, dt), torch.randn(R * C, device=dev).to(tdt))
    y = tpp.TensorView(tpp.TensorDesc(C, R, C, dt), torch.empty(R * C, device=dev, dtype=tdt))
    es = x.primary.element_size()
    timeit(lambda: transform(x, TransformSpec(TransformKind.TRANSPOSE), y), 2 * R * C * es, f"TRANSPOSE {dt.name} {R}x{C}")
xb = tpp.TensorView(tpp.TensorDesc(R, C, R, tpp.DType.BF16), torch.randn(R * C, device=dev).to(torch.bfloat16))
yv = tpp.TensorView(tpp.TensorDesc(R * 2, C // 2, R * 2, tpp.DType.BF16), torch.empty(R * C, device=dev, dtype=torch.bfloat16))
timeit(lambda: transform(xb, TransformSpec(TransformKind.VNNI, alpha=2), yv), 2 * R * C * 2, f"VNNI bf16 {R}x{C}")
yt = tpp.TensorView(tpp.TensorDesc(C * 2, R // 2, C * 2, tpp.DType.BF16), torch.empty(R * C, device=dev, dtype=torch.bfloat16))
timeit(lambda: transform(yv, TransformSpec(TransformKind.VNNI_TO_VNNIT, alpha=2, alpha_out=2, rows=R, cols=C), yt), 2 * R * C * 2, f"VNNI_TO_VNNIT bf16 {R}x{C}")
a = tpp.TensorView(tpp.TensorDesc(R, C, R, tpp.DType.BF16), torch.randn(R * C, device=dev).to(torch.bfloat16))
o = tpp.TensorView(tpp.TensorDesc(R, C, R, tpp.DType.BF16), torch.empty(R * C, device=dev, dtype=torch.bfloat16))
timeit(lambda: tpp.apply_unary(tpp.UnaryKind.RELU, a, o), 2 * R * C * 2, f"RELU bf16 {R}x{C}")
timeit(lambda: tpp.apply_binary(tpp.BinaryKind.ADD, a, a, o), 3 * R * C * 2, f"ADD bf16 {R}x{C}")
