"""Per-tile timestamps (%globaltimer) of CTA 0 in one tensor-core launch:
stage0-full (MMA side), last MMA issued, accumulator ready (epilogue), TMEM
slot released.  Diagnostics only: python tools/tile_ts.py [conv|fc]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_05755_b200 as tpp
from paper_2104_05755_b200 import _lib

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(0)
lib = _lib.load()
buf = torch.zeros(400, dtype=torch.int64, device=dev)
which = sys.argv[1] if len(sys.argv) > 1 else "conv"
if which == "conv":
    spec = tpp.ConvSpec(256, 1, 1, 56, 56)
    xin = torch.rand(256 * 56 * 56 * 64, generator=gen, device=dev).to(torch.bfloat16)
    wv = (torch.randn(9 * 64 * 64, generator=gen, device=dev) * 0.1).to(torch.bfloat16)
    conv = tpp.Conv2d(spec, wv)
    yo = torch.empty_like(xin)
    fn = lambda: conv.forward(xin, out=yo)
else:
    layer, x, out = bench.make_fc_set(torch, tpp, gen, dev, 512, 16, 32, 64, 64, 64, tpp.UnaryKind.GELU, 1.0, 0.02,
                                      bias=False)
    fn = lambda: layer.forward(x, 512, 32, out=out)
for it in range(2):
    buf.zero_()
    lib.tpp_debug_phase_timestamps(buf.data_ptr())
    g = bench.graph_of(torch, [fn] * 5)
    lib.tpp_debug_phase_timestamps(None)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    t = buf.cpu().tolist()
    print(f"{which}: per launch {e0.elapsed_time(e1) * 1e3 / 5:.2f} us; exit at {(t[6] - t[0]) / 1e3:.2f}")
    prev = None
    for k in range(32):
        f, m, a, r = t[16 + 4 * k: 20 + 4 * k]
        if f == 0:
            break
        z = lambda v: (v - t[0]) / 1e3 if v else float("nan")
        print(f"  tile {k:2d}: load_issued {z(t[200 + k]):7.2f}  tempty_ok {z(t[240 + k]):7.2f}"
              f"  full {z(f):7.2f}  mma_done {z(m):7.2f}  acc_ready {z(a):7.2f}  released {z(r):7.2f}"
              f"  epi {(r - a) / 1e3 if a and r else float('nan'):5.2f}  mma {(m - f) / 1e3:5.2f}")
    # epilogue chunk stamps of tile 4 (warp 4): after tcgen05.ld, after activation, after pack, after store issue
    base = t[16 + 4 * 4 + 2]
    if base:
        for ch in range(8):
            v = t[150 + 4 * ch: 154 + 4 * ch]
            if not v[0]:
                break
            print(f"    chunk {ch}: " + " ".join(f"{(x - base) / 1e3:6.2f}" if x else "   nan" for x in v))

    z = lambda v: (v - t[0]) / 1e3 if v else float("nan")
    for w in range(8):
        print(f"  tile 20 epilogue warp {w}: acc_ready {z(t[300 + w]):7.2f}  tmem_released {z(t[280 + w]):7.2f}  done {z(t[290 + w]):7.2f}")
    if t[320] and t[322]:
        print(f"  SM clock over tiles 4..30 (CTA 0): {(t[322] - t[320]) / (t[323] - t[321]) * 1e3:.0f} MHz")
