"""Phase timestamps (%globaltimer, CTA 0) of one FC tensor-core launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_05755_b200 as tpp
from paper_2104_05755_b200 import _lib
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(0)
lib = _lib.load()
buf = torch.zeros(16, dtype=torch.int64, device=dev)
names = ["start", "prologue", "stage0 landed", "last MMA issued", "acc ready", "epilogue done", "exit", "tmem ld done", "stores issued", "-", "wait released", "first TMA issued"]
import ctypes as C
def fwd_flags(layer, x, nb, bn, out, extra):
    d = layer.desc(nb, bn, _lib.FC_BIAS | extra)
    _lib.check(lib.tpp_fc_forward(C.byref(d), layer.w_packed.data_ptr(), x.data_ptr(), layer.bias.data_ptr(), None,
                                  out.data_ptr(), None, _lib.stream_ptr()))
for label, (nb, cb, kb, bn, bnt, extra) in {"cfg2": (16, 16, 16, 64, 64, 0), "K=64": (16, 1, 16, 64, 64, 0), "big": (64, 16, 16, 64, 64, 0)}.items():
    layer, x, out = bench.make_fc_set(torch, tpp, gen, dev, nb, cb, bn, 64, kb, 64, tpp.UnaryKind.RELU, 0.02, 0.02)
    layer.forward = (lambda l, e: (lambda x, nb, bn, out: fwd_flags(l, x, nb, bn, out, e)))(layer, extra)
    for it in range(2):
        # stamps of the LAST launch of a graph of 20 back-to-back launches (clocks up)
        lib.tpp_debug_phase_timestamps(buf.data_ptr())
        g = bench.graph_of(torch, [lambda: layer.forward(x, nb, bn, out=out)] * 20)
        lib.tpp_debug_phase_timestamps(None)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        t = buf.cpu().tolist()
        print(label, f"per launch {e0.elapsed_time(e1)*1e3/20:.2f} us |", " ".join(f"{n}={(v - t[0])/1e3:.2f}" for n, v in zip(names, t[:12])))
