"""Benchmark of the B200 TPP BRGEMM hot path (driver contract: one JSON line).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
blocked BF16 fully-connected layer, N = C = K = 1024, bn = bc = bk = 64,
bias + ReLU fused, FP32 accumulation — one `FcLayer.forward` (one tcgen05
BRGEMM launch) per step.  Synthetic normal(0, 0.02) data.

* ``value``   — whole-job TFLOP/s, inputs resident in HBM; each timed region
  is EXACTLY K steps (CUDA graph of K launches) bracketed by barrier +
  synchronize; the per-step input/weight/output sets rotate through > 2x L2
  (126 MB) of buffers so no step hits a warm L2.  Max over ranks.
* ``e2e``     — the same layer through the public API with HOST buffers:
  pinned H2D of the step's input, forward, D2H of the output, every step.
* ``roofline``— dominant kernel (brgemm_tc_kernel) vs the measured bf16
  burst peak in MEASURED_PEAKS.json.
* ``cpu_baseline`` — the CPU oracle port (numpy restatement of the
  reference, oracle/tpp_oracle.py) on a bounded sample, rank 0 only.
* ``extra``   — the other BASELINE configs measured the same way (FFN + LN,
  conv fwd / bwd-data, LN alone, cfg-1 BRGEMM) for the roofline tables.

``--impl reference`` times the reference algorithm (the oracle port; the
Python reference itself cannot travel to the GPU box) on all host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# cfg 2 (BASELINE naming: tokens N = Nb*bn, in-channels C = Cb*bc, out K = Kb*bk)
NB, CB, BN, BC, KB, BK = 16, 16, 64, 64, 16, 64
FLOPS_CFG2 = 2 * (NB * BN) * (CB * BC) * (KB * BK)
METRIC = "BRGEMM-layer TFLOP/s & % bf16 tensor peak; eltwise TPP GB/s & % HBM peak"
L2_BYTES = 126 * 1024 * 1024


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d["bf16_tflops"], d.get("bf16_tflops_sustained"), d["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# synthetic data (BASELINE cfg 2: all values normal(0, 0.02))
# ---------------------------------------------------------------------------

def _vnni_from_logical(wl):
    """[Kb][Cb][bk][bc] logical weight blocks -> VNNI-2 [Kb][Cb][bc/2][bk][2]."""
    kb, cb, bk, bc = wl.shape
    return wl.reshape(kb, cb, bk, bc // 2, 2).permute(0, 1, 3, 2, 4).contiguous()


def make_fc_set(torch, tpp, gen, dev, n_b, c_b, bn, bc, k_b, bk, act, std_x, std_w, bias=True):
    x = (torch.randn(n_b * c_b * bn * bc, generator=gen, device=dev) * std_x).to(torch.bfloat16)
    wl = (torch.randn(k_b, c_b, bk, bc, generator=gen, device=dev) * std_w).to(torch.bfloat16)
    b = (torch.randn(k_b * bk, generator=gen, device=dev) * std_w).to(torch.bfloat16) if bias else None
    layer = tpp.FcLayer(k_b, c_b, bk, bc, _vnni_from_logical(wl).reshape(-1), bias=b, activation=act)
    out = torch.empty(n_b * k_b * bn * bk, dtype=torch.bfloat16, device=dev)
    return layer, x, out


def graph_of(torch, fns):
    """Capture a list of launch closures into one CUDA graph."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in fns:  # warm (lazy attribute setup) outside capture
            f()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for f in fns:
            f()
    torch.cuda.synchronize()
    return g


def time_graph(torch, dist, g, reps_min=5, min_seconds=1.0):
    """Replay a K-step graph repeatedly; each replay is one timed region
    (barrier + sync both sides, CUDA events on the launching stream).
    Returns per-replay milliseconds (max over ranks)."""
    times = []
    t_start = time.perf_counter()
    while len(times) < reps_min or time.perf_counter() - t_start < min_seconds:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        times.append(ms)
        if len(times) > 2000:
            break
    return times


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args, rank, world, dist):
    import numpy as np
    import torch

    import paper_2104_05755_b200 as tpp

    dev = torch.device("cuda", torch.cuda.current_device())
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    K, W = args.steps, args.warmup
    peak_bf16, peak_bf16_sus, peak_hbm, peak_src = _peaks()
    relu = tpp.UnaryKind.RELU

    # ---- rotating cfg-2 sets, > 2x L2 in total -----------------------------
    set_bytes = (NB * CB * BN * BC + KB * CB * BK * BC + NB * KB * BN * BK) * 2
    n_sets = max(2, min(K, (2 * L2_BYTES) // set_bytes + 1))
    sets = [make_fc_set(torch, tpp, gen, dev, NB, CB, BN, BC, KB, BK, relu, 0.02, 0.02)
            for _ in range(n_sets)]
    torch.cuda.synchronize()

    def step_fn(i):
        layer, x, out = sets[i % n_sets]
        return lambda: layer.forward(x, NB, BN, out=out)

    g_warm = graph_of(torch, [step_fn(i) for i in range(max(W, 1))])
    for _ in range(3):
        g_warm.replay()
    g = graph_of(torch, [step_fn(i) for i in range(K)])
    dev_index = torch.cuda.current_device()
    with ClockSampler(dev_index) as cs:
        times = time_graph(torch, dist, g, min_seconds=1.0)
    clocks = cs.summary()
    ms_region = statistics.median(times)
    ms_step = ms_region / K
    value = FLOPS_CFG2 * world / (ms_step * 1e-3) / 1e12
    kernel_tflops = FLOPS_CFG2 / (ms_step * 1e-3) / 1e12

    # ---- e2e through the public API with host buffers ------------------------
    layer0, x0, _ = sets[0]
    n_in = NB * CB * BN * BC
    n_out = NB * KB * BN * BK
    x_host = torch.empty(n_in, dtype=torch.bfloat16, pin_memory=True)
    x_host.copy_(x0.cpu())
    # NBUF-deep buffering: H2D of step i only waits for compute of step
    # i - NBUF and compute of step i only for the D2H of step i - NBUF.  (The
    # step time is the PCIe link: 66-68 us with 2 or 4 buffers, eager or
    # graph-captured; tools/copy_overlap.py: H2D 44.6, D2H 41.0, both
    # directions concurrently 49-53 us per 2 MiB pair.)
    NBUF = 4
    out_host = [torch.empty(n_out, dtype=torch.bfloat16, pin_memory=True) for _ in range(NBUF)]
    x_dev = [torch.empty(n_in, dtype=torch.bfloat16, device=dev) for _ in range(NBUF)]
    out_dev = [torch.empty(n_out, dtype=torch.bfloat16, device=dev) for _ in range(NBUF)]
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(NBUF)]
    ev_comp = [torch.cuda.Event() for _ in range(NBUF)]
    ev_out = [torch.cuda.Event() for _ in range(NBUF)]
    for e in ev_comp + ev_out:
        e.record(comp)

    def e2e_step(i, comp):
        """Pipelined serving step: H2D of step i overlaps compute of i-1 and
        the D2H of earlier steps (NBUF-deep device and host buffers, 3 streams)."""
        b = i % NBUF
        with torch.cuda.stream(s_in):
            if i >= NBUF:
                s_in.wait_event(ev_comp[b])      # x_dev[b] no longer read
            x_dev[b].copy_(x_host, non_blocking=True)
            ev_in[b].record(s_in)
        comp.wait_event(ev_in[b])
        if i >= NBUF:
            comp.wait_event(ev_out[b])           # out_dev[b] already copied out
        layer0.forward(x_dev[b], NB, BN, out=out_dev[b], stream=comp)
        ev_comp[b].record(comp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_comp[b])
            out_host[b].copy_(out_dev[b], non_blocking=True)
            ev_out[b].record(s_out)

    # the K-step serving loop is captured once as a CUDA graph (copies, the
    # layer's kernel and the cross-stream events), then replayed: per step the
    # timed region still moves the step's input H2D and its output D2H
    def e2e_graph():
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            cap = torch.cuda.current_stream()
            s_in.wait_stream(cap)
            s_out.wait_stream(cap)
            for i in range(K):
                e2e_step(i, cap)
            cap.wait_stream(s_in)
            cap.wait_stream(s_out)
        return gr

    for i in range(max(W, 3)):
        e2e_step(i, comp)
    torch.cuda.synchronize()
    g_e2e = e2e_graph()
    # the copy engines / PCIe link take a few hundred ms of traffic to reach
    # steady state: warm the serving graph before timing it
    t_w = time.perf_counter()
    while time.perf_counter() - t_w < 0.5:
        g_e2e.replay()
        torch.cuda.synchronize()
    e2e_times = []
    for _ in range(15):
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        g_e2e.replay()
        e1.record(comp)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        e2e_times.append(ms)
    if os.environ.get("TPP_BENCH_DEBUG"):
        print("e2e region ms:", e2e_times, file=sys.stderr)
    e2e_ms_step = statistics.median(e2e_times) / K
    e2e_value = FLOPS_CFG2 * world / (e2e_ms_step * 1e-3) / 1e12

    # the other configs and the CPU baseline are single-GPU reports (N = 1 runs)
    extra = {}
    if rank == 0 and world == 1 and not args.no_extra:
        extra = run_extra(args, torch, tpp, dev, gen, peak_bf16, peak_hbm)

    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("brgemm_tc_kernel_cfg2_bytes_per_launch")
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_sample()

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "TFLOP/s",
            "n_gpus": world,
            "steps": K,
            "warmup": W,
            "ms_per_step": round(ms_step, 6),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic normal(0,0.02), seeded; weights random-init",
            "config": {
                "workload": "cfg2: blocked BF16 FC fwd N=C=K=1024 (bn=bc=bk=64) + bias + ReLU, fp32 acc",
                "global_batch": NB * BN * world,
                "per_gpu_tokens": NB * BN,
                "parallelism": f"dp{world} (minibatch shards, no collective)",
                "l2": f"rotating {n_sets} input/weight/output sets ({n_sets * set_bytes / 2**20:.0f} MiB > 2x L2)",
                "timing": f"median of {len(times)} CUDA-graph replays of exactly K={K} steps",
            },
            "roofline": {
                "bound": "tensor",
                "achieved": round(kernel_tflops, 2),
                "peak": peak_bf16,
                "unit": "TFLOP/s",
                "frac": round(kernel_tflops / peak_bf16, 4),
                "traffic": traffic,
                "kernel": "brgemm_tc_kernel<BN=64> (tcgen05 + TMA, bias+ReLU fused)",
                "algorithmic_flops_per_launch": FLOPS_CFG2,
                "peak_source": f"bf16_tflops burst, {peak_src}",
            },
            "e2e": {
                "value": round(e2e_value, 3),
                "unit": "TFLOP/s",
                "h2d_bytes_per_step": n_in * 2,
                "d2h_bytes_per_step": n_out * 2,
                "ms_per_step": round(e2e_ms_step, 6),
                "api": "FcLayer.forward with a pinned H2D of the input and a D2H of the output every step; copies pipelined against compute on separate streams (4-deep buffers), the K-step serving loop captured once as a CUDA graph and replayed",
            },
            "gpu_launches": K,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "extra": extra,
        }
        print(json.dumps(line), flush=True)


def run_extra(args, torch, tpp, dev, gen, peak_bf16, peak_hbm):
    """Other BASELINE configs, same timing method (CUDA graph of R steps,
    rotating buffers where the working set is smaller than L2)."""
    out = {}
    R = 20
    # ---- cfg 3: BERT-large FFN + LayerNorm (T=16384, bn=32, bc=bk=64) -----
    try:
        nb, bn, h, f = 512, 32, 16, 64   # 1024 hidden = 16 blocks, 4096 = 64 blocks
        x = (torch.randn(nb * h * bn * 64, generator=gen, device=dev)).to(torch.bfloat16)
        w1 = (torch.randn(f, h, 64, 64, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
        w2 = (torch.randn(h, f, 64, 64, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
        fc1 = tpp.FcLayer(f, h, 64, 64, _vnni_from_logical(w1).reshape(-1), activation=tpp.UnaryKind.GELU)
        fc2 = tpp.FcLayer(h, f, 64, 64, _vnni_from_logical(w2).reshape(-1))
        mid = torch.empty(nb * f * bn * 64, dtype=torch.bfloat16, device=dev)
        o2 = torch.empty(nb * h * bn * 64, dtype=torch.bfloat16, device=dev)
        ln = torch.empty_like(o2)
        gam = torch.ones(1024, device=dev)
        bet = torch.zeros(1024, device=dev)
        fl1 = 2 * 16384 * 1024 * 4096
        parts = {
            "fc1_gelu": lambda: fc1.forward(x, nb, bn, out=mid),
            "fc2_residual": lambda: fc2.forward(mid, nb, bn, out=o2, residual=x),
            "layernorm": lambda: tpp.layernorm_blocked(o2, nb, h, bn, 64, 1e-5, gam, bet, out=ln),
        }
        res = {}
        total = 0.0
        for name, fn in parts.items():
            g = graph_of(torch, [fn] * R)
            ms = statistics.median(time_graph(torch, None, g, reps_min=5, min_seconds=0.3)) / R
            total += ms
            if name == "layernorm":
                byts = 2 * 16384 * 1024 * 2
                res[name] = {"ms": round(ms, 5), "GB/s": round(byts / ms / 1e6, 1),
                             "frac_hbm": round(byts / ms / 1e6 / peak_hbm, 4),
                             "parity": "bitwise vs oracle in tests/test_gpu_parity.py"}
            else:
                tf = fl1 / ms / 1e9
                res[name] = {"ms": round(ms, 5), "TFLOP/s": round(tf, 1),
                             "frac_bf16": round(tf / peak_bf16, 4)}
        res["ffn_step_ms"] = round(total, 5)
        res["ffn_TFLOP/s"] = round(2 * fl1 / total / 1e9, 1)
        # LayerNorm in the tolerance mode (tree-ordered sums, FMA scaling)
        g = graph_of(torch, [lambda: tpp.layernorm_blocked(o2, nb, h, bn, 64, 1e-5, gam, bet, out=ln,
                                                           exact=False)] * R)
        ms = statistics.median(time_graph(torch, None, g, reps_min=5, min_seconds=0.3)) / R
        byts = 2 * 16384 * 1024 * 2
        res["layernorm_tolerance_mode"] = {"ms": round(ms, 5), "GB/s": round(byts / ms / 1e6, 1),
                                           "frac_hbm": round(byts / ms / 1e6 / peak_hbm, 4),
                                           "parity": "statistics <= 1e-5 rel. of the exact path, "
                                                     "outputs within the BF16 tolerance (tests)"}
        out["cfg3_bert_ffn_ln"] = res
        del x, w1, w2, fc1, fc2, mid, o2, ln
    except Exception as e:  # keep the headline line even if an extra fails
        out["cfg3_bert_ffn_ln"] = {"error": str(e)[:200]}
    # ---- cfg 4: ResNet conv 3x3, N=256, C=K=64, 56x56 -----------------------
    try:
        spec = tpp.ConvSpec(256, 1, 1, 56, 56)
        xin = torch.rand(256 * 56 * 56 * 64, generator=gen, device=dev).to(torch.bfloat16)
        wl = (torch.randn(1, 1, 3, 3, 64, 64, generator=gen, device=dev) * (2 / 576) ** 0.5).to(torch.bfloat16)
        wv = wl.reshape(1, 1, 3, 3, 64, 32, 2).permute(0, 1, 2, 3, 5, 4, 6).contiguous().reshape(-1)
        conv = tpp.Conv2d(spec, wv)
        yo = torch.empty_like(xin)
        dO = torch.randn(256 * 56 * 56 * 64, generator=gen, device=dev).to(torch.bfloat16)
        dI = torch.empty_like(xin)
        res = {}
        byts = 2 * 256 * 56 * 56 * 64 * 2 + 9 * 64 * 64 * 2
        dW = torch.empty(9 * 64 * 64, dtype=torch.float32, device=dev)
        for name, fn in (("fwd", lambda: conv.forward(xin, out=yo)),
                         ("bwd_data", lambda: conv.backward_data(dO, din=dI)),
                         ("bwd_weights", lambda: conv.backward_weights(xin, dO, dw=dW))):
            g = graph_of(torch, [fn] * 5)
            ms = statistics.median(time_graph(torch, None, g, reps_min=5, min_seconds=0.3)) / 5
            tf = spec.flops / ms / 1e9
            res[name] = {"ms": round(ms, 5), "TFLOP/s": round(tf, 1), "frac_bf16": round(tf / peak_bf16, 4),
                         "GB/s": round(byts / ms / 1e6, 1), "frac_hbm": round(byts / ms / 1e6 / peak_hbm, 4)}
        out["cfg4_conv3x3"] = res
        del xin, yo, dO, dI, conv, dW
    except Exception as e:
        out["cfg4_conv3x3"] = {"error": str(e)[:200]}
    # ---- cfg 5: 4-layer blocked MLP training step (fwd + CE + bwd + split-SGD), 1 GPU ----
    try:
        dims = [1024, 4096, 4096, 4096, 1024]
        tokens = 8192
        mlp = tpp.BlockedMLP(dims, tokens, bn=64, lr=0.01, device=dev, seed=7)
        xin = torch.randn(tokens * 1024, generator=gen, device=dev).to(torch.bfloat16)
        tg = torch.randint(0, 1024, (tokens,), generator=gen, device=dev, dtype=torch.int32)
        g = graph_of(torch, [lambda: mlp.train_step(xin, tg)] * 3)
        ms = statistics.median(time_graph(torch, None, g, reps_min=5, min_seconds=0.5)) / 3
        tf = mlp.flops_per_step / ms / 1e9
        out["cfg5_mlp_train_step"] = {"ms": round(ms, 4), "TFLOP/s": round(tf, 1),
                                      "frac_bf16_sustained": round(tf / 1409.7, 4),
                                      "flops_per_step": mlp.flops_per_step,
                                      "loss_mean": round(float(mlp.loss.mean()), 4)}
        del mlp, xin, tg
    except Exception as e:
        out["cfg5_mlp_train_step"] = {"error": str(e)[:200]}
    # ---- standalone memory-bound TPPs (dense BF16 8192 x 4096 views) ---------
    # three rotating operand sets (3 x 128 MiB > 2x L2): every launch streams HBM
    try:
        from paper_2104_05755_b200.ops import TransformKind, TransformSpec, transform
        R, Cc = 8192, 4096
        mk = lambda rows, cols: tpp.TensorView(tpp.TensorDesc(rows, cols, rows, tpp.DType.BF16),  # noqa: E731
                                               torch.randn(rows * cols, generator=gen, device=dev).to(torch.bfloat16))
        sets_ = [(mk(R, Cc), mk(R, Cc), mk(R, Cc)) for _ in range(3)]
        trs = [mk(Cc, R) for _ in range(3)]
        vns = [mk(2 * R, Cc // 2) for _ in range(3)]
        nb = R * Cc * 2
        cases = {
            "relu": (lambda k: tpp.apply_unary(tpp.UnaryKind.RELU, sets_[k][0], sets_[k][1]), 2 * nb),
            "add": (lambda k: tpp.apply_binary(tpp.BinaryKind.ADD, sets_[k][0], sets_[k][1], sets_[k][2]), 3 * nb),
            "transpose": (lambda k: transform(sets_[k][0], TransformSpec(TransformKind.TRANSPOSE), trs[k]), 2 * nb),
            "vnni": (lambda k: transform(sets_[k][0], TransformSpec(TransformKind.VNNI, alpha=2), vns[k]), 2 * nb),
            "vnni_to_vnnit": (lambda k: transform(vns[k], TransformSpec(TransformKind.VNNI_TO_VNNIT, alpha=2,
                                                                        alpha_out=2, rows=R, cols=Cc),
                                                  sets_[k][2]), 2 * nb),
            # per-column xorshift128 draws + mask + scaled copy (bitwise the reference)
            "dropout": (lambda k: tpp.apply_unary(tpp.UnaryKind.DROPOUT, sets_[k][0], sets_[k][1],
                                                  dropout_p=0.1), 2 * nb + R * Cc // 8),
            "dropout_inv": (lambda k: tpp.apply_unary(tpp.UnaryKind.DROPOUT_INV, sets_[k][0], sets_[k][2],
                                                      dropout_p=0.1), 2 * nb + R * Cc // 8),
        }
        for k in range(3):
            sets_[k][0].tertiary = {"prng": tpp.PrngState(k, Cc)}
            sets_[k][0].secondary = torch.zeros(R * Cc // 8, dtype=torch.uint8, device=dev)
        res = {}
        for name, (fn, byts) in cases.items():
            g = graph_of(torch, [(lambda k=k: fn(k)) for k in range(3)] * 2)
            ms = statistics.median(time_graph(torch, None, g, reps_min=5, min_seconds=0.2)) / 6
            res[name] = {"us": round(ms * 1e3, 2), "GB/s": round(byts / ms / 1e6, 1),
                         "frac_hbm": round(byts / ms / 1e6 / peak_hbm, 4)}
        res["shape"] = "bf16 8192 x 4096 column-major views (transforms: 8192 x 4096 logical)"
        out["memory_bound_tpps"] = res
        del sets_, trs, vns
    except Exception as e:
        out["memory_bound_tpps"] = {"error": str(e)[:200]}
    # ---- INT8 BRGEMM on tcgen05 kind::i8 (exact: integer sums) -------------------
    try:
        m = n = 4096
        k, cnt = 1024, 8
        a = torch.randint(-128, 128, (cnt * k * m,), generator=gen, device=dev, dtype=torch.int8)
        b = torch.randint(-128, 128, (cnt * n * k,), generator=gen, device=dev, dtype=torch.int8)
        cs = [tpp.alloc(tpp.TensorDesc(m, n, m, tpp.DType.INT32), device=dev) for _ in range(2)]
        spec8 = tpp.GemmSpec(m, n, k, m, k, m, in_dtype=tpp.DType.INT8, out_dtype=tpp.DType.INT32)
        batch8 = tpp.BrgemmBatch.stride(a, b, k * m, n * k, cnt)
        g = graph_of(torch, [lambda: tpp.brgemm(spec8, batch8, cs[0]), lambda: tpp.brgemm(spec8, batch8, cs[1])] * 2)
        ms = statistics.median(time_graph(torch, None, g, reps_min=5, min_seconds=0.3)) / 4
        tops = 2.0 * m * n * k * cnt / ms / 1e9
        out["int8_brgemm_tc"] = {"shape": "M=N=4096, K=1024, STRIDE batch of 8", "ms": round(ms, 4),
                                 "TOPS": round(tops, 1), "frac_nominal_int8_dense": round(tops / 4500.0, 4),
                                 "parity": "bitwise (integer sums) vs the reference in tests/test_gpu_parity.py"}
        del a, b, cs
    except Exception as e:
        out["int8_brgemm_tc"] = {"error": str(e)[:200]}
    # ---- cfg 1: FP32 BRGEMM 16 x 64^3, beta = 1, reference order (bitwise) ------
    try:
        m = n = k = 64
        a = torch.rand(m * k * 16, generator=gen, device=dev) * 2 - 1
        b = torch.rand(k * n * 16, generator=gen, device=dev) * 2 - 1
        c = tpp.TensorView(tpp.TensorDesc(m, n, m, tpp.DType.FP32), torch.rand(m * n, generator=gen, device=dev))
        spec1 = tpp.GemmSpec(m, n, k, m, k, m, beta=1.0)
        batch = tpp.BrgemmBatch.stride(a, b, m * k, k * n, 16)
        g = graph_of(torch, [lambda: tpp.brgemm(spec1, batch, c)] * R)
        ms = statistics.median(time_graph(torch, None, g, reps_min=5, min_seconds=0.2)) / R
        out["cfg1_brgemm_fp32_ordered"] = {"latency_us": round(ms * 1e3, 2),
                                           "GFLOP/s": round(8388608 / ms / 1e6, 1),
                                           "parity": "bitwise vs oracle in tests/test_gpu_parity.py"}
    except Exception as e:
        out["cfg1_brgemm_fp32_ordered"] = {"error": str(e)[:200]}
    return out


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port (numpy restatement of the reference)
# ---------------------------------------------------------------------------

def _cfg2_host_inputs(seed=0):
    import numpy as np
    from oracle import tpp_oracle as O
    rng = np.random.default_rng(seed)
    x = O.fp32_to_bf16_rne(rng.normal(0, 0.02, (NB, CB, BN, BC)).astype(np.float32))
    wl = O.fp32_to_bf16_rne(rng.normal(0, 0.02, (KB, CB, BK, BC)).astype(np.float32))
    wv = wl.reshape(KB, CB, BK, BC // 2, 2).transpose(0, 1, 3, 2, 4).copy()
    b = O.fp32_to_bf16_rne(rng.normal(0, 0.02, KB * BK).astype(np.float32))
    return x, wv, b


def cpu_baseline_sample():
    """Single-thread oracle port on the full cfg-2 workload (~3 s)."""
    from oracle import tpp_oracle as O
    x, wv, b = _cfg2_host_inputs()
    t0 = time.perf_counter()
    O.fc_forward_bf16(x, wv, b, activation="relu")
    dt = time.perf_counter() - t0
    return {"value": round(FLOPS_CFG2 / dt / 1e12, 8), "unit": "TFLOP/s", "cores": 1,
            "kind": "port",
            "sample": f"full cfg2 workload (1024x1024x1024 BF16 FC + bias + ReLU) once, "
                      f"{dt:.2f} s, oracle/tpp_oracle.py fc_forward_bf16 (numpy, reference order)"}


_REF_STATE = {}


def _ref_init(seed):
    _REF_STATE["inputs"] = _cfg2_host_inputs(seed)


def _ref_block(nb):
    from oracle import tpp_oracle as O
    x, wv, b = _REF_STATE["inputs"]
    out, _, _ = O.fc_forward_bf16(x, wv, b, activation="relu", nb_sel=[nb])
    return int(out.view("uint16").sum() % 65521)


def run_reference(args, rank, world):
    """The reference algorithm on the host: the oracle port over all cores,
    each step = the full cfg-2 workload (16 token blocks over a process pool)."""
    if rank != 0:
        return
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    procs = max(1, min(cores, NB))
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_ref_init, initargs=(0,)) as pool:
        for _ in range(max(args.warmup, 1)):
            pool.map(_ref_block, range(NB))
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_ref_block, range(NB))
        dt = (time.perf_counter() - t0) / args.steps
    val = FLOPS_CFG2 * world / dt / 1e12
    line = {
        "metric": METRIC, "value": round(val, 8), "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic normal(0,0.02), seeded",
        "config": {"workload": "cfg2: blocked BF16 FC fwd N=C=K=1024 (bn=bc=bk=64) + bias + ReLU, fp32 acc",
                   "global_batch": NB * BN * world, "parallelism": f"{procs} host processes"},
        "impl": "reference",
        "cpu_baseline": {"value": round(val, 8), "unit": "TFLOP/s", "cores": procs, "kind": "port",
                         "sample": f"full cfg2 workload per step over {procs} processes "
                                   f"(oracle/tpp_oracle.py, the reference's per-element order)"},
        "e2e": {"value": round(val, 8), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = dist_mod
    run_ours(args, rank, world, dist)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
