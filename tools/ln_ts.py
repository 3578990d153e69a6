"""Per-group timestamps of CTA 0 in the TMA LayerNorm (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_05755_b200 as tpp
from paper_2104_05755_b200 import _lib
dev = torch.device("cuda", 0)
lib = _lib.load()
buf = torch.zeros(600, dtype=torch.int64, device=dev)
x = torch.randn(16384 * 1024, device=dev).to(torch.bfloat16)
o = torch.empty_like(x)
gam = torch.ones(1024, device=dev) if os.environ.get("LN_AFFINE") else None
bet = torch.zeros(1024, device=dev) if os.environ.get("LN_AFFINE") else None
fn = lambda: tpp.layernorm_blocked(x, 512, 16, 32, 64, 1e-5, gam, bet, out=o,
                                   exact=os.environ.get("LN_EXACT", "1") == "1")
NL = int(os.environ.get("NL", "3"))
for it in range(2):
    buf.zero_()
    lib.tpp_debug_phase_timestamps(buf.data_ptr())
    g = bench.graph_of(torch, [fn] * NL)
    lib.tpp_debug_phase_timestamps(None)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    t = buf.cpu().tolist()
    print(f"per launch {e0.elapsed_time(e1) * 1e3 / NL:.2f} us")
    z = lambda v: f"{(v - t[0]) / 1e3:6.2f}" if v else "   -  "
    for i in range(16):
        v = t[8 + 5 * i: 13 + 5 * i]
        if not any(v):
            break
        print(f"  group {i:2d}: load {z(v[0])} fold {z(v[1])}..{z(v[2])} applied {z(v[3])} stored {z(v[4])}")
    st = [(t[200 + 2 * b] - t[0]) / 1e3 for b in range(148)]
    en = [(t[201 + 2 * b] - t[0]) / 1e3 for b in range(148)]
    import statistics as S
    print(f"  CTA start min/med/max {min(st):.2f}/{S.median(st):.2f}/{max(st):.2f}  end min/med/max {min(en):.2f}/{S.median(en):.2f}/{max(en):.2f}")
    print("  latest CTAs:", sorted(range(148), key=lambda b: -en[b])[:8], [round(en[b], 2) for b in sorted(range(148), key=lambda b: -en[b])[:8]])
    res = [(t[500 + b] - t[0]) / 1e3 for b in range(64)]
    print(f"  CTA resident (before griddepcontrol.wait) min/med/max {min(res):.2f}/{S.median(res):.2f}/{max(res):.2f}")
