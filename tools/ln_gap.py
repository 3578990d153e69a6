"""Gap between consecutive LayerNorm launches: last CTA exit of launch A vs
first CTA residency / wait release of launch B (absolute %globaltimer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05755_b200 as tpp
from paper_2104_05755_b200 import _lib
dev = torch.device("cuda", 0)
lib = _lib.load()
x = torch.randn(16384 * 1024, device=dev).to(torch.bfloat16)
o = torch.empty_like(x)
bufs = [torch.zeros(600, dtype=torch.int64, device=dev) for _ in range(3)]
exact = os.environ.get("LN_EXACT", "1") == "1"
fn = lambda: tpp.layernorm_blocked(x, 512, 16, 32, 64, 1e-5, out=o, exact=exact)
for _ in range(3):
    fn()
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for b in bufs:
        lib.tpp_debug_phase_timestamps(b.data_ptr())
        fn()
    lib.tpp_debug_phase_timestamps(None)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
t = [b.cpu().tolist() for b in bufs]
for i in range(3):
    st = [t[i][200 + 2 * c] for c in range(148)]
    en = [t[i][201 + 2 * c] for c in range(148)]
    res = [t[i][500 + c] for c in range(64)]
    base = min(res)
    print(f"launch {i}: resident {(min(res)-base)/1e3:.2f}..{(max(res)-base)/1e3:.2f}  start {(min(st)-base)/1e3:.2f}..{(max(st)-base)/1e3:.2f}"
          f"  end {(min(en)-base)/1e3:.2f}..{(max(en)-base)/1e3:.2f}")
    if i:
        prev_end = max(t[i - 1][201 + 2 * c] for c in range(148))
        print(f"   gap: prev last end -> first resident {(min(res) - prev_end)/1e3:.2f} us, -> first start {(min(st) - prev_end)/1e3:.2f} us")
