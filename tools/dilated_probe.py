"""Time the ATACworks-scale dilated conv1d (W=60400, Q=60000, C=K=15, S=51,
d=8, FP32) through dilated_conv1d_forward; with TPP_ORDERED_NO_COLS=1 set the
generic ordered tile kernel runs instead of the column kernel."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05755_b200 as tpp

C = K = 15; S = 51; d = 8; Q = 60000; W = Q + (S - 1) * d
g = torch.Generator(device="cuda").manual_seed(0)
x = tpp.TensorView(tpp.TensorDesc(C, W, C, tpp.DType.FP32), torch.rand(C * W, generator=g, device="cuda"))
w = tpp.TensorView(tpp.TensorDesc(C * S, K, C * S, tpp.DType.FP32), torch.rand(C * S * K, generator=g, device="cuda"))
o = tpp.TensorView(tpp.TensorDesc(K, Q, K, tpp.DType.FP32), torch.empty(K * Q, device="cuda"))
spec = tpp.DilatedConvSpec(C, K, W, Q, S, d)
for _ in range(3):
    tpp.dilated_conv1d_forward(spec, x, w, o)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); tpp.dilated_conv1d_forward(spec, x, w, o); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
fl = 2.0 * C * K * S * Q
print(f"dilated conv: {ms*1e3:.1f} us  {fl/ms/1e6:.1f} GFLOP/s")
