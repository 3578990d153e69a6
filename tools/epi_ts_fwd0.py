"""Epilogue chunk clocks (clock64, CTA 0, warp 4) of one tile of the cfg-5
fwd0 GEMM (8192 tokens x 1024 -> 4096, ReLU + mask; the CTA-pair kernel) in a
TPP_PHASE_STAMPS build: per 32-column chunk, cycles after the accumulator was
ready at chunk start / math done / packed / store issued."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05755_b200 as tpp
from paper_2104_05755_b200 import _lib
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(0)
lib = _lib.load()
TOK = 8192
bf = lambda n, s=1.0: (torch.randn(n, generator=g, device=dev) * s).to(torch.bfloat16)
L0 = tpp.FcLayer(64, 16, 64, 64, None, activation=tpp.UnaryKind.RELU, w_packed=bf(4096 * 1024, 0.02))
x0 = bf(TOK * 1024)
o0 = torch.empty(TOK * 4096, dtype=torch.bfloat16, device=dev)
m0 = torch.empty(TOK * 4096 // 8, dtype=torch.uint8, device=dev)
buf = torch.zeros(512, dtype=torch.int64, device=dev)
for it in range(3):
    L0.forward(x0, TOK // 64, 64, out=o0, relu_mask=m0)
for it in range(2):
    buf.zero_()
    lib.tpp_debug_phase_timestamps(buf.data_ptr())
    L0.forward(x0, TOK // 64, 64, out=o0, relu_mask=m0)
    lib.tpp_debug_phase_timestamps(None)
    torch.cuda.synchronize()
    t = buf.cpu().tolist()
    base = t[189]
    print("tile", os.environ.get("TPP_DBG_TILE", "0"), "ld issued", t[188] - base)
    for ch in range(8):
        s = t[150 + 4 * ch: 154 + 4 * ch]
        if s[0]:
            print(f"  chunk {ch}: start={s[0]-base} math={s[1]-base} packed={s[2]-base} issued={s[3]-base}")
    # tile start stamps of CTA 0 (gtimer ns) for the first tiles
    t0 = t[16]
    for i in range(8):
        a = t[16 + 4 * i: 20 + 4 * i]
        if a[0]:
            print(f"  tile {i}: mma first issue={a[0]-t0} ns, mma committed={a[1]-t0}, epi acc ready={a[2]-t0}, epi done={a[3]-t0}; producer tile start={t[200+i]-t0 if t[200+i] else None}")
