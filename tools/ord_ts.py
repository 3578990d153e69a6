"""Phase stamps of the staged ordered BRGEMM (cfg 1), diagnostics."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_05755_b200 as tpp
from paper_2104_05755_b200 import _lib
dev = torch.device("cuda", 0)
lib = _lib.load()
buf = torch.zeros(16, dtype=torch.int64, device=dev)
m = n = k = 64
A = torch.rand(m * k * 16, device=dev); B = torch.rand(k * n * 16, device=dev)
c = tpp.TensorView(tpp.TensorDesc(m, n, m, tpp.DType.FP32), torch.rand(m * n, device=dev))
sp = tpp.GemmSpec(m, n, k, m, k, m, beta=1.0)
bt = tpp.BrgemmBatch.stride(A, B, m * k, k * n, 16)
fn = lambda: tpp.brgemm(sp, bt, c)
for it in range(3):
    lib.tpp_debug_phase_timestamps(buf.data_ptr())
    g = bench.graph_of(torch, [fn] * 10)
    lib.tpp_debug_phase_timestamps(None)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    t = buf.cpu().tolist()
    print(f"per launch {e0.elapsed_time(e1) * 1e3 / 10:.2f} us; staged {(t[1]-t[0])/1e3:.2f} us, computed {(t[2]-t[1])/1e3:.2f} us")
