"""Benchmark of the B200 TPP BRGEMM hot path (driver contract: one JSON line).

Headline workload = BASELINE.json configs[4] (cfg 5), the largest config that
fits one GPU and the only one with a collective: one training step of the
blocked BF16 MLP 1024 -> 4096 -> 4096 -> 4096 -> 1024 (ReLU, no bias), global
minibatch 8192 tokens (bn = 64): forward (4 tcgen05 BRGEMM layers, ReLU +
bitmask fused), softmax cross-entropy gradient, backward-weights and
backward-data BRGEMMs (RELU_INV fused), split-SGD on FP32 masters.  At N GPUs
the global batch is sharded over the minibatch (8192/N tokens per rank,
strong scaling) and every dW bucket is sum-allreduced over NCCL on a side
stream (BF16 buckets at N > 1) with that layer's split-SGD right behind it.

* ``value``    — whole-job TFLOP/s (global-batch step flops / step time);
  N = 1: each timed region is a CUDA graph of EXACTLY K steps; N > 1: K eager
  steps; barrier + synchronize on both sides, CUDA events, max over ranks.
  The step's working set (~1 GB) is far larger than L2: every step streams
  its weights and activations from HBM.
* ``e2e``      — the same step through the public API (``BlockedMLP.train_step``)
  with HOST buffers: pinned H2D of the step's tokens and targets, D2H of the
  per-token loss, every step; eager (headline) and graph-replayed.
* ``roofline`` — the dominant kernel: the CTA-pair tcgen05 BRGEMM
  (``brgemm_tc_kernel<256,3,2,0,2,1>``) over the six 4096 x 4096 GEMMs of the
  step, timed with CUDA events on its launching stream inside a K-step
  breakdown pass, against the measured bf16 burst peak (MEASURED_PEAKS.json;
  the sustained-peak fraction is reported beside it).
* ``cpu_baseline`` — the oracle port of the reference (oracle/tpp_oracle.py,
  the reference's per-element order) on a bounded sample of the same step
  (64 tokens through all four full-size layers), rank 0, N = 1.
* ``extra``    — the other BASELINE configs the same way (cfg 2 FC, cfg 3 FFN
  + LN, cfg 4 conv, cfg 1 BRGEMM), BRGEMM per addressing variant, memory-
  bound TPPs, INT8; at N > 1 the per-N compute / allreduce / exposed-
  communication breakdown and an allreduce size sweep.

``--impl reference`` times the reference algorithm on the host (the oracle
port: the Python reference cannot travel to the GPU box) over all cores.
``--gpus N`` outside torchrun spawns N ranks itself (torch.distributed.run).
``--dry-run`` exercises the multi-rank plumbing on CPU (gloo), no GPU.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIMS = [1024, 4096, 4096, 4096, 1024]
GLOBAL_TOKENS = 8192
TOK_BLOCK = 64
LR = 0.01
METRIC = "BRGEMM-layer TFLOP/s & % bf16 tensor peak; eltwise TPP GB/s & % HBM peak"
WORKLOAD = ("cfg5: blocked BF16 MLP 1024-4096-4096-4096-1024 training step (fwd + softmax-CE + "
            "bwd-data + bwd-weights + split-SGD), global batch 8192 tokens sharded over the "
            "minibatch, bn=64, fp32 accumulation")
L2_BYTES = 126 * 1024 * 1024
# cfg 2 (BASELINE naming: tokens N = Nb*bn, in-channels C = Cb*bc, out K = Kb*bk)
NB, CB, BN, BC, KB, BK = 16, 16, 64, 64, 16, 64
FLOPS_CFG2 = 2 * (NB * BN) * (CB * BC) * (KB * BK)


def cfg5_flops(tokens: int, dims=DIMS) -> int:
    """fwd + dW (same) + dX of layers 2..4 (the first layer's dX is not needed)."""
    fwd = sum(2 * tokens * dims[l] * dims[l + 1] for l in range(len(dims) - 1))
    dx = sum(2 * tokens * dims[l] * dims[l + 1] for l in range(1, len(dims) - 1))
    return 2 * fwd + dx


FLOPS_CFG5 = cfg5_flops(GLOBAL_TOKENS)   # 1,992,864,825,344


def bench_config(world: int) -> dict:
    """Identical in both arms (the driver compares the dicts)."""
    return {"workload": WORKLOAD, "global_batch": GLOBAL_TOKENS, "per_gpu_tokens": GLOBAL_TOKENS // world,
            "dims": DIMS, "bn": TOK_BLOCK, "lr": LR}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"burst": d["bf16_tflops"], "sustained": d.get("bf16_tflops_sustained") or d["bf16_tflops"],
                "hbm": d["hbm_gbs"], "src": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"burst": 1590.0, "sustained": 1400.0, "hbm": 6650.0, "src": "fallback (B200_PROFILING.md)"}


def _cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


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
# timing helpers
# ---------------------------------------------------------------------------

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


def _max_over_ranks(torch, dist, ms: float) -> float:
    if dist is None:
        return ms
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


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
        times.append(_max_over_ranks(torch, dist, e0.elapsed_time(e1)))
        if len(times) > 2000:
            break
    return times


def time_eager(torch, dist, fn, K, reps=5, tail=None):
    """K eager calls per timed region (barrier + sync both sides, CUDA events
    on the current stream, max over ranks); ``tail`` (e.g. joining deferred
    updates) runs inside the region after the K calls."""
    times = []
    for _ in range(reps):
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            fn()
        if tail is not None:
            tail()
        e1.record()
        torch.cuda.synchronize()
        times.append(_max_over_ranks(torch, dist, e0.elapsed_time(e1)))
    return times


# ---------------------------------------------------------------------------
# our arm: cfg 5 training step
# ---------------------------------------------------------------------------

def step_breakdown(torch, mlp, x, tg, steps):
    """Per-launch device time inside K eager steps: a CUDA event is recorded
    on the main stream right after every launch (BlockedMLP.trace), so each
    interval is one kernel (serialised: an event between two kernels ends
    their programmatic-dependent-launch overlap, so the sum slightly exceeds
    the graph-replayed step)."""
    recs = []

    def tr(label):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        recs[-1].append((label, ev))

    mlp.trace = tr
    try:
        for _ in range(steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
            recs.append([("start", e0)])
            mlp.train_step(x, tg)
    finally:
        mlp.trace = None
    torch.cuda.synchronize()
    per = {}
    for rec in recs:
        for (_, a), (lab, b) in zip(rec[:-1], rec[1:]):
            per.setdefault(lab, []).append(a.elapsed_time(b))
    return {lab: statistics.median(v) for lab, v in per.items()}


def count_kernels(torch, fn):
    """Kernels one call of ``fn`` launches, by name (torch.profiler / CUPTI)."""
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        names = {}
        for e in prof.events():
            if getattr(e, "device_type", None) is not None and "CUDA" in str(e.device_type):
                n = e.name.split("(")[0]
                if n.startswith("void "):
                    n = n[5:]
                if not n.startswith("tpp::"):  # only this library's kernels (not copies / collectives)
                    continue
                names[n] = names.get(n, 0) + 1
        return names
    except Exception as ex:  # profiler unavailable: caller falls back to the static count
        return {"error": str(ex)[:120]}


def run_e2e(torch, tpp, mlp, dist, K, W, graph: bool):
    """BlockedMLP.train_step with host buffers: per step a pinned H2D of the
    step's tokens (BF16) and targets (int32) on a copy stream (double
    buffered, overlapping the previous step), and a D2H of the per-token loss
    into pinned memory.  Returns (ms per step, h2d bytes, d2h bytes)."""
    dev = mlp.device
    tokens = mlp.tokens
    n_x = tokens * DIMS[0]
    gen = torch.Generator()
    gen.manual_seed(99)
    x_host = torch.randn(n_x, generator=gen).to(torch.bfloat16).pin_memory()
    t_host = torch.randint(0, DIMS[-1], (tokens,), generator=gen, dtype=torch.int32).pin_memory()
    NBUF = 2
    loss_host = [torch.empty(tokens, dtype=torch.float32).pin_memory() for _ in range(NBUF)]
    x_dev = [torch.empty(n_x, dtype=torch.bfloat16, device=dev) for _ in range(NBUF)]
    t_dev = [torch.empty(tokens, dtype=torch.int32, device=dev) for _ in range(NBUF)]
    s_in = torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(NBUF)]
    ev_done = [torch.cuda.Event() for _ in range(NBUF)]
    comp0 = torch.cuda.current_stream()
    for e in ev_done:
        e.record(comp0)

    def step(i, comp, capturing=False):
        b = i % NBUF
        with torch.cuda.stream(s_in):
            if not (capturing and i < NBUF):       # (a capture may not wait on pre-capture work)
                s_in.wait_event(ev_done[b])        # buffers b no longer read
            x_dev[b].copy_(x_host, non_blocking=True)
            t_dev[b].copy_(t_host, non_blocking=True)
            ev_in[b].record(s_in)
        comp.wait_event(ev_in[b])
        loss = mlp.train_step(x_dev[b], t_dev[b])
        loss_host[b].copy_(loss, non_blocking=True)
        ev_done[b].record(comp)

    for i in range(max(W, 3)):
        step(i, comp0)
    mlp.sync_updates()   # a capture must not depend on the eager steps' deferred updates
    torch.cuda.synchronize()
    if graph:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            cap = torch.cuda.current_stream()
            s_in.wait_stream(cap)
            for i in range(K):
                step(i, cap, capturing=True)
            mlp.sync_updates()
            cap.wait_stream(s_in)
        torch.cuda.synchronize()
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        times = time_graph(torch, dist, gr, reps_min=5, min_seconds=0.5)
    else:
        ctr = [0]

        def one():
            step(ctr[0], torch.cuda.current_stream())
            ctr[0] += 1

        times = time_eager(torch, dist, one, K, reps=5, tail=mlp.sync_updates)
    return statistics.median(times) / K, n_x * 2 + tokens * 4, tokens * 4


def run_ours(args, rank, world, dist):
    import torch

    import paper_2104_05755_b200 as tpp
    from paper_2104_05755_b200 import parallel

    dev = torch.device("cuda", torch.cuda.current_device())
    K, W = args.steps, args.warmup
    peaks = _peaks()
    tokens = GLOBAL_TOKENS // world
    grad_dtype = args.grad_dtype or ("fp32" if world == 1 else "bf16")
    # one rank: the backward overlaps dW_l with dX_{l-1} on a side stream and
    # the next step's layer-0 GEMM runs beside the last updates (defer_join);
    # every timed region ends by joining them (sync_updates)
    mlp = tpp.BlockedMLP(DIMS, tokens, bn=TOK_BLOCK, lr=LR, global_batch=GLOBAL_TOKENS, seed=7, device=dev,
                         grad_dtype=grad_dtype, defer_join=True)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    x = torch.randn(tokens * DIMS[0], generator=gen, device=dev).to(torch.bfloat16)
    tg = torch.randint(0, DIMS[-1], (tokens,), generator=gen, device=dev, dtype=torch.int32)
    step = lambda: mlp.train_step(x, tg)  # noqa: E731
    for _ in range(W):
        step()
    mlp.sync_updates()
    torch.cuda.synchronize()

    # ---- headline: K training steps per timed region -----------------------
    use_graph = world == 1 and not args.eager
    with ClockSampler(torch.cuda.current_device()) as cs:
        if use_graph:
            g = graph_of(torch, [step] * K + [mlp.sync_updates])
            g.replay()
            torch.cuda.synchronize()
            times = time_graph(torch, None, g, reps_min=5, min_seconds=1.0)
        else:
            times = time_eager(torch, dist, step, K, reps=max(5, args.reps), tail=mlp.sync_updates)
    clocks = cs.summary()
    ms_step = statistics.median(times) / K
    value = FLOPS_CFG5 / (ms_step * 1e-3) / 1e12
    loss_mean = float(mlp.loss.mean())

    # ---- per-launch breakdown and the dominant kernel ----------------------
    bd = step_breakdown(torch, mlp, x, tg, K)
    big = [lab for lab in bd if mlp.gemm_flops(lab) and DIMS[int(lab[-1])] == 4096 and DIMS[int(lab[-1]) + 1] == 4096]
    dom_ms = sum(bd[lab] for lab in big)
    dom_flops = sum(mlp.gemm_flops(lab) for lab in big)
    dom_tf = dom_flops / (dom_ms * 1e-3) / 1e12 if dom_ms > 0 else 0.0
    gemm_ms = sum(v for lab, v in bd.items() if mlp.gemm_flops(lab))
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("pair_kernel_fwd_4096x4096x8192_bytes_per_launch")
        except Exception:
            traffic = None
    kern = count_kernels(torch, step)
    launches_per_step = sum(v for k, v in kern.items() if k != "error") if "error" not in kern else 16

    # ---- e2e through the public API ----------------------------------------
    e2e_ms, h2d, d2h = run_e2e(torch, tpp, mlp, dist, K, W, graph=False)
    e2e_graph_ms = None
    if world == 1:
        e2e_graph_ms, _, _ = run_e2e(torch, tpp, mlp, dist, K, W, graph=True)

    # ---- N > 1: compute vs communication -----------------------------------
    scaling = None
    if world > 1:
        real_sync = mlp.sync
        mlp.sync = parallel.GradSync(reduce_fn=lambda t: None, device=dev)  # same streams, no collective
        for _ in range(2):
            step()
        comp_ms = statistics.median(time_eager(torch, dist, step, K, reps=3)) / K
        mlp.sync = real_sync
        el = 2 if grad_dtype == "bf16" else 4
        sweep = parallel.allreduce_sweep([DIMS[l] * DIMS[l + 1] * el for l in range(len(DIMS) - 1)],
                                         dtype=torch.bfloat16 if el == 2 else torch.float32)
        scaling = {"compute_only_ms_per_step": round(comp_ms, 4), "step_ms": round(ms_step, 4),
                   "exposed_comm_ms": round(ms_step - comp_ms, 4),
                   "allreduce_ms_per_bucket": {str(k): round(v, 4) for k, v in sweep.items()},
                   "allreduce_ms_total": round(sum(sweep.values()), 4),
                   "grad_dtype": grad_dtype}

    extra = {}
    if rank == 0 and world == 1 and not args.no_extra:
        extra = run_extra(args, torch, tpp, dev, gen, peaks)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_sample()

    comm = None
    if world > 1:
        comm = {"backend": dist.get_backend(), "nranks": dist.get_world_size(),
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                "one_gpu_functional_check": os.environ.get("TPP_BENCH_ONE_GPU") == "1",
                "high_priority_streams": True, "nccl_init_log": _nccl_init_lines()}
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
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic: tokens normal(0,1), weights normal(0,0.02) random-init, targets uniform [0,1024), seeded",
            "config": bench_config(world),
            "parallelism": (f"dp{world}: {tokens} tokens per rank; " +
                            ("no collective" if world == 1 else
                             f"per-layer {grad_dtype} dW sum-allreduce (NCCL) on a side stream, split-SGD behind each bucket")),
            "l2": "step working set ~1 GB (weights, masters, activations, gradients) >> 126 MB L2: every step streams HBM",
            "timing": (f"median of {len(times)} CUDA-graph replays of exactly K={K} steps" if use_graph
                       else f"median of {len(times)} regions of K={K} eager steps, max over ranks"),
            "loss_mean": round(loss_mean, 5),
            "roofline": {
                "bound": "tensor",
                "achieved": round(dom_tf, 2),
                "peak": peaks["burst"],
                "unit": "TFLOP/s",
                "frac": round(dom_tf / peaks["burst"], 4),
                "traffic": traffic,
                "kernel": "brgemm_tc_kernel<256,3,2,0,2,1> (tcgen05 cta_group::2, TMA ring, epilogue fused) "
                          "over the six 4096x4096 GEMMs of the step (fwd, bwd-data, bwd-weights)",
                "algorithmic_flops_per_step": dom_flops,
                "kernel_ms_per_step": round(dom_ms, 5),
                "share_of_step": round(dom_ms / ms_step, 4),
                "frac_of_sustained": round(dom_tf / peaks["sustained"], 4),
                "peak_source": f"bf16_tflops burst (the conservative denominator: the breakdown pass is a "
                               f"short {K}-step run), {peaks['src']}; sustained {peaks['sustained']}",
                "traffic_note": "dram read+write of one forward launch of the kernel (ncu --set full, "
                                "profiles/r2_ncu_pair_fwd.txt); algorithmic 171,966,464 B",
                "step_frac_of_sustained": round(value / world / peaks["sustained"], 4),
            },
            "step_breakdown_ms": {k: round(v, 5) for k, v in bd.items()},
            "step_breakdown_sum_ms": round(sum(bd.values()), 5),
            "gemm_ms_per_step": round(gemm_ms, 5),
            "e2e": {
                "value": round(FLOPS_CFG5 / (e2e_ms * 1e-3) / 1e12, 3),
                "unit": "TFLOP/s",
                "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "ms_per_step": round(e2e_ms, 6),
                "graph_replayed": (None if e2e_graph_ms is None else
                                   {"value": round(FLOPS_CFG5 / (e2e_graph_ms * 1e-3) / 1e12, 3),
                                    "ms_per_step": round(e2e_graph_ms, 6)}),
                "api": "BlockedMLP.train_step (eager) with a pinned H2D of the step's tokens + targets on a copy "
                       "stream (double-buffered) and a D2H of the per-token loss every step",
            },
            "gpu_launches": K * launches_per_step,
            "kernels_per_step": kern,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "comm": comm,
            "scaling_breakdown": scaling,
            "extra": extra,
        }
        print(json.dumps(line), flush=True)


def _nccl_init_lines():
    path = os.environ.get("NCCL_DEBUG_FILE", "")
    lines = []
    try:
        import glob
        for fn in glob.glob(path.replace("%h", "*").replace("%p", "*")):
            with open(fn) as f:
                for ln in f:
                    if "nranks" in ln or "NVLS" in ln or "comm " in ln:
                        lines.append(ln.strip()[-160:])
    except Exception:
        pass
    return lines[:8]


def run_extra(args, torch, tpp, dev, gen, peaks):
    """Other BASELINE configs, same timing method (CUDA graph of R steps,
    rotating buffers where the working set is smaller than L2)."""
    peak_bf16, peak_hbm = peaks["burst"], peaks["hbm"]
    peak_sus = peaks["sustained"]   # the extras replay for >= 0.3 s: the clock settles under the power cap
    out = {}
    R = 20
    relu = tpp.UnaryKind.RELU
    # ---- cfg 2: blocked BF16 FC 1024^3 + bias + ReLU (rotating sets > 2x L2) --
    try:
        set_bytes = (NB * CB * BN * BC + KB * CB * BK * BC + NB * KB * BN * BK) * 2
        n_sets = max(2, (2 * L2_BYTES) // set_bytes + 1)
        sets = []
        for _ in range(n_sets):
            xx = (torch.randn(NB * CB * BN * BC, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
            wl = (torch.randn(KB, CB, BK, BC, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
            bb = (torch.randn(KB * BK, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
            layer = tpp.FcLayer(KB, CB, BK, BC, _vnni_from_logical(wl).reshape(-1), bias=bb, activation=relu)
            sets.append((layer, xx, torch.empty(NB * KB * BN * BK, dtype=torch.bfloat16, device=dev)))
        fns = [(lambda s=s: s[0].forward(s[1], NB, BN, out=s[2])) for s in sets]
        g = graph_of(torch, (fns * (R // len(fns) + 1))[:R])
        ms = statistics.median(time_graph(torch, None, g, reps_min=5, min_seconds=0.5)) / R
        tf = FLOPS_CFG2 / ms / 1e9
        out["cfg2_fc_bias_relu"] = {"us": round(ms * 1e3, 3), "TFLOP/s": round(tf, 1),
                                    "frac_bf16_burst": round(tf / peak_bf16, 4),
                                    "frac_bf16_sustained": round(tf / peak_sus, 4),
                                    "l2": f"{n_sets} rotating sets > 2x L2"}
        del sets, fns, g
    except Exception as e:
        out["cfg2_fc_bias_relu"] = {"error": str(e)[:200]}
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
                             "parity": "bitwise vs oracle (tests/test_gpu_dispatch.py::test_cfg3_chain_full_size)"}
            else:
                tf = fl1 / ms / 1e9
                res[name] = {"ms": round(ms, 5), "TFLOP/s": round(tf, 1),
                             "frac_bf16": round(tf / peak_bf16, 4), "frac_bf16_sustained": round(tf / peak_sus, 4)}
        res["ffn_step_ms"] = round(total, 5)
        res["ffn_TFLOP/s"] = round(2 * fl1 / total / 1e9, 1)
        g = graph_of(torch, [lambda: tpp.layernorm_blocked(o2, nb, h, bn, 64, 1e-5, gam, bet, out=ln,
                                                           exact=False)] * R)
        ms = statistics.median(time_graph(torch, None, g, reps_min=5, min_seconds=0.3)) / R
        byts = 2 * 16384 * 1024 * 2
        res["layernorm_tolerance_mode"] = {"ms": round(ms, 5), "GB/s": round(byts / ms / 1e6, 1),
                                           "frac_hbm": round(byts / ms / 1e6 / peak_hbm, 4)}
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
                         "frac_bf16_sustained": round(tf / peak_sus, 4),
                         "GB/s": round(byts / ms / 1e6, 1), "frac_hbm": round(byts / ms / 1e6 / peak_hbm, 4)}
        out["cfg4_conv3x3"] = res
        del xin, yo, dO, dI, conv, dW
    except Exception as e:
        out["cfg4_conv3x3"] = {"error": str(e)[:200]}
    # ---- BRGEMM TPP through brgemm(): BF16 per addressing variant ------------
    try:
        out["brgemm_bf16_tcgen05"] = brgemm_variants(torch, tpp, dev, gen, peak_bf16)
    except Exception as e:
        out["brgemm_bf16_tcgen05"] = {"error": str(e)[:200]}
    # ---- standalone memory-bound TPPs (dense BF16 8192 x 4096 views) ---------
    # three rotating operand sets (3 x 128 MiB > 2x L2): every launch streams HBM
    try:
        from paper_2104_05755_b200.ops import TransformKind, TransformSpec, transform
        Rr, Cc = 8192, 4096
        mk = lambda rows, cols: tpp.TensorView(tpp.TensorDesc(rows, cols, rows, tpp.DType.BF16),  # noqa: E731
                                               torch.randn(rows * cols, generator=gen, device=dev).to(torch.bfloat16))
        sets_ = [(mk(Rr, Cc), mk(Rr, Cc), mk(Rr, Cc)) for _ in range(3)]
        trs = [mk(Cc, Rr) for _ in range(3)]
        vns = [mk(2 * Rr, Cc // 2) for _ in range(3)]
        nb = Rr * Cc * 2
        cases = {
            "relu": (lambda k: tpp.apply_unary(tpp.UnaryKind.RELU, sets_[k][0], sets_[k][1]), 2 * nb),
            "add": (lambda k: tpp.apply_binary(tpp.BinaryKind.ADD, sets_[k][0], sets_[k][1], sets_[k][2]), 3 * nb),
            "transpose": (lambda k: transform(sets_[k][0], TransformSpec(TransformKind.TRANSPOSE), trs[k]), 2 * nb),
            "vnni": (lambda k: transform(sets_[k][0], TransformSpec(TransformKind.VNNI, alpha=2), vns[k]), 2 * nb),
            "vnni_to_vnnit": (lambda k: transform(vns[k], TransformSpec(TransformKind.VNNI_TO_VNNIT, alpha=2,
                                                                        alpha_out=2, rows=Rr, cols=Cc),
                                                  sets_[k][2]), 2 * nb),
            "dropout": (lambda k: tpp.apply_unary(tpp.UnaryKind.DROPOUT, sets_[k][0], sets_[k][1],
                                                  dropout_p=0.1), 2 * nb + Rr * Cc // 8),
            "dropout_inv": (lambda k: tpp.apply_unary(tpp.UnaryKind.DROPOUT_INV, sets_[k][0], sets_[k][2],
                                                      dropout_p=0.1), 2 * nb + Rr * Cc // 8),
        }
        for k in range(3):
            sets_[k][0].tertiary = {"prng": tpp.PrngState(k, Cc)}
            sets_[k][0].secondary = torch.zeros(Rr * Cc // 8, dtype=torch.uint8, device=dev)
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
                                 "TOPS": round(tops, 1),
                                 "note": "no measured INT8 peak on this pool (MEASURED_PEAKS has bf16 only); "
                                         "2x the measured bf16 burst would be the dense int8 analogue",
                                 "frac_of_2x_measured_bf16_burst": round(tops / (2 * peak_bf16), 4),
                                 "parity": "bitwise (integer sums) vs the reference in tests/test_gpu_parity.py"}
        del a, b, cs
    except Exception as e:
        out["int8_brgemm_tc"] = {"error": str(e)[:200]}
    # ---- 1-D dilated conv at the paper's ATACworks scale (address/stride BRGEMM user) ----
    try:
        C_, K_, S_, d_, Q_ = 15, 15, 51, 8, 60000
        W_ = Q_ + (S_ - 1) * d_
        spec_d = tpp.DilatedConvSpec(C_, K_, W_, Q_, S_, d_)
        inp = tpp.TensorView(tpp.TensorDesc(C_, W_, C_, tpp.DType.FP32),
                             torch.randn(C_ * W_, generator=gen, device=dev))
        wv = tpp.TensorView(tpp.TensorDesc(C_ * S_, K_, C_ * S_, tpp.DType.FP32),
                            torch.randn(C_ * S_ * K_, generator=gen, device=dev))
        outd = tpp.alloc(tpp.TensorDesc(K_, Q_, K_, tpp.DType.FP32), device=dev)
        g = graph_of(torch, [lambda: tpp.dilated_conv1d_forward(spec_d, inp, wv, outd)] * 5)
        ms = statistics.median(time_graph(torch, None, g, reps_min=5, min_seconds=0.3)) / 5
        fl = 2 * C_ * K_ * S_ * Q_
        simt = 148 * 128 * 2 * 1.965e9 / 1e12   # FP32 SIMT peak (TFLOP/s), SURVEY §8(d)
        out["dilated_conv1d_atacworks"] = {
            "shape": "W=60400, Q=60000, C=K=15, S=51, d=8, FP32 (PAPER.md:819)", "us": round(ms * 1e3, 2),
            "GFLOP/s": round(fl / ms / 1e6, 1), "frac_fp32_simt_peak": round(fl / ms / 1e9 / simt, 4),
            "frac_no_fma_bound": round(2 * fl / ms / 1e9 / simt, 4),
            "kernel": "K1w brgemm_ordered_window_kernel (bitwise order: separate mul + add, so half the FMA peak)",
            "parity": "bitwise vs the reference order (tests/test_gpu_parity.py)"}
        del inp, wv, outd
    except Exception as e:
        out["dilated_conv1d_atacworks"] = {"error": str(e)[:200]}
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


def _vnni_from_logical(wl):
    """[Kb][Cb][bk][bc] logical weight blocks -> VNNI-2 [Kb][Cb][bc/2][bk][2]."""
    kb, cb, bk, bc = wl.shape
    return wl.reshape(kb, cb, bk, bc // 2, 2).permute(0, 1, 3, 2, 4).contiguous()


def brgemm_variants(torch, tpp, dev, gen, peak_bf16):
    """BF16 BRGEMM through the reference API (Engine.AUTO -> tcgen05 K11)
    per addressing variant: the cfg-2 composition (256 C blocks of 64 x 64,
    16 VNNI weight blocks x input blocks each, kernels.py:312-329) issued as
    ONE brgemm_grouped launch per variant; plus a single large brgemm()
    (one C block of 1024 x 1024, 16 reduce blocks of 64)."""
    Nb, Cb, bn, bc, Kb, bk = 16, 16, 64, 64, 16, 64
    blk = bc * bk
    R = 20
    n_sets = 4          # rotating operand sets so repeated launches do not just hit L2
    res = {}
    spec = tpp.GemmSpec(bk, bn, bc, bk, bc, bk, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32,
                        a_layout=tpp.ALayout.VNNI)
    groups = [(nb, kb) for nb in range(Nb) for kb in range(Kb)]
    coffs = [(nb * Kb + kb) * bn * bk for nb, kb in groups]
    sets = []
    for _ in range(n_sets):
        x = torch.randn(Nb * Cb * blk, generator=gen, device=dev).to(torch.bfloat16)
        w = (torch.randn(Kb * Cb * blk, generator=gen, device=dev) * 0.02).to(torch.bfloat16)
        out = torch.empty(Nb * Kb * bn * bk, dtype=torch.float32, device=dev)
        sets.append((x, w, out))
    for variant in ("stride", "offset", "address"):
        fns = []
        for x, w, out in sets:
            if variant == "stride":
                gb = tpp.GroupedBatch.stride(w, x, blk, blk, Cb, [kb * Cb * blk for _, kb in groups],
                                             [nb * Cb * blk for nb, _ in groups])
            elif variant == "offset":
                gb = tpp.GroupedBatch.offset(w, x, [[(kb * Cb + i) * blk for i in range(Cb)] for _, kb in groups],
                                             [[(nb * Cb + i) * blk for i in range(Cb)] for nb, _ in groups])
            else:
                gb = tpp.GroupedBatch.address([[(w, (kb * Cb + i) * blk) for i in range(Cb)] for _, kb in groups],
                                              [[(x, (nb * Cb + i) * blk) for i in range(Cb)] for nb, _ in groups])
            fns.append(lambda gb=gb, out=out: tpp.brgemm_grouped(spec, gb, out, coffs))
        g = graph_of(torch, (fns * R)[:R])
        from paper_2104_05755_b200 import _lib
        ms = statistics.median(time_graph(torch, None, g, reps_min=5, min_seconds=0.3)) / R
        tf = FLOPS_CFG2 / ms / 1e9
        res[f"cfg2_composition_{variant}"] = {"us": round(ms * 1e3, 3), "TFLOP/s": round(tf, 1),
                                              "frac_bf16_burst": round(tf / peak_bf16, 4),
                                              "kernel": _lib.last_config()}
    # one large C block: brgemm() with a 1024 x 1024 x (16 x 64) STRIDE batch
    m = n = 1024
    k, cnt = 64, 16
    a = (torch.randn(cnt * m * k, generator=gen, device=dev)).to(torch.bfloat16)
    b = (torch.randn(cnt * k * n, generator=gen, device=dev)).to(torch.bfloat16)
    c = tpp.TensorView(tpp.TensorDesc(m, n, m, tpp.DType.FP32), torch.empty(m * n, device=dev))
    sp = tpp.GemmSpec(m, n, k, m, k, m, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32)
    bt = tpp.BrgemmBatch.stride(a, b, m * k, k * n, cnt)
    g = graph_of(torch, [lambda: tpp.brgemm(sp, bt, c)] * R)
    ms = statistics.median(time_graph(torch, None, g, reps_min=5, min_seconds=0.3)) / R
    tf = 2 * m * n * k * cnt / ms / 1e9
    from paper_2104_05755_b200 import _lib
    res["single_brgemm_1024x1024_stride16"] = {"us": round(ms * 1e3, 3), "TFLOP/s": round(tf, 1),
                                                "frac_bf16_burst": round(tf / peak_bf16, 4),
                                                "kernel": _lib.last_config(), "a_layout": "plain (MN-major)"}
    res["parity"] = "normwise <= 2e-2 vs the reference (tests/test_gpu_brgemm_tc.py)"
    return res


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port (numpy restatement of the reference)
# ---------------------------------------------------------------------------

SAMPLE_TOKENS = 64


def _cfg5_host_inputs(tokens, seed=0):
    import numpy as np
    from oracle import tpp_oracle as O
    rng = np.random.default_rng(seed)
    ws = [rng.standard_normal((DIMS[l + 1], DIMS[l]), dtype=np.float32) * np.float32(0.02)
          for l in range(len(DIMS) - 1)]
    x = O.fp32_to_bf16_rne(rng.standard_normal((tokens, DIMS[0]), dtype=np.float32))
    tg = rng.integers(0, DIMS[-1], tokens).astype(np.int32)
    return ws, x, tg


def cpu_baseline_sample():
    """Single-thread oracle port: one training step of the full-size MLP on a
    64-token sample (fwd + CE + bwd-data + bwd-weights + split-SGD), ~16 s."""
    from oracle import tpp_oracle as O
    ws, x, tg = _cfg5_host_inputs(SAMPLE_TOKENS)
    t0 = time.perf_counter()
    O.mlp_train_step(x, ws, tg, LR, GLOBAL_TOKENS)
    dt = time.perf_counter() - t0
    return {"value": round(cfg5_flops(SAMPLE_TOKENS) / dt / 1e12, 8), "unit": "TFLOP/s", "cores": 1,
            "kind": "port", "cpu_model": _cpu_model(),
            "sample": f"cfg5 training step on {SAMPLE_TOKENS} of the 8192 tokens through all four full-size "
                      f"layers ({cfg5_flops(SAMPLE_TOKENS) / 1e9:.2f} GFLOP) in {dt:.2f} s, "
                      f"oracle/tpp_oracle.py mlp_train_step (numpy, the reference's per-element order); "
                      f"throughput extrapolates linearly in tokens"}


_REF = {}


def _ref_init(seed):
    import numpy as np
    from oracle import tpp_oracle as O
    ws, x, tg = _cfg5_host_inputs(SAMPLE_TOKENS, seed)
    _REF["w"] = [O.bf16_to_fp32((w.view(np.uint32) >> 16).astype(np.uint16)) for w in ws]
    rng = np.random.default_rng(seed + 1)
    _REF["h"] = [O.round_bf16(np.abs(rng.standard_normal((SAMPLE_TOKENS, DIMS[l]), dtype=np.float32)))
                 for l in range(len(DIMS) - 1)]
    _REF["g"] = [O.round_bf16(rng.standard_normal((SAMPLE_TOKENS, DIMS[l + 1]), dtype=np.float32) * np.float32(1e-4))
                 for l in range(len(DIMS) - 1)]


def _ref_layer(l):
    """One layer's share of a training step on 64 tokens in the reference
    order: forward, backward-weights, backward-data (layers 2-4)."""
    from oracle import tpp_oracle as O
    w, h, g = _REF["w"][l], _REF["h"][l], _REF["g"][l]
    z = O.blocked_matmul(h, w)
    dw = O.blocked_matmul(g.T.copy(), h.T.copy())
    flops = 2 * 2 * SAMPLE_TOKENS * DIMS[l] * DIMS[l + 1]
    if l > 0:
        O.blocked_matmul(g, w.T.copy())
        flops += 2 * SAMPLE_TOKENS * DIMS[l] * DIMS[l + 1]
    return flops, float(z[0, 0] + dw[0, 0])


def run_reference(args, rank, world):
    """The reference algorithm on the host: the oracle port over all cores.
    One step = every process runs one layer's fwd + bwd-weights + bwd-data
    on a 64-token sample (layers assigned round-robin, so a step covers all
    four layer shapes); value = flops done / step wall time."""
    if rank != 0:
        return
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    procs = max(1, min(cores, 16))
    ctx = mp.get_context("fork")
    layers = [p % (len(DIMS) - 1) for p in range(procs)]
    with ctx.Pool(procs, initializer=_ref_init, initargs=(0,)) as pool:
        n_warm = max(1, min(args.warmup, 3))   # each CPU step is seconds long: at most 3 warm-ups
        for _ in range(n_warm):
            pool.map(_ref_layer, layers)
        t0 = time.perf_counter()
        flops = 0
        for _ in range(args.steps):
            flops += sum(f for f, _ in pool.map(_ref_layer, layers))
        dt = time.perf_counter() - t0
    val = flops / dt / 1e12
    line = {
        "metric": METRIC, "value": round(val, 8), "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": n_warm, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: tokens normal(0,1), weights normal(0,0.02) random-init, targets uniform [0,1024), seeded",
        "config": bench_config(world),
        "impl": "reference",
        "parallelism": f"{procs} host processes",
        "cpu_baseline": {"value": round(val, 8), "unit": "TFLOP/s", "cores": procs, "kind": "port",
                         "cpu_model": _cpu_model(),
                         "sample": f"per step {procs} processes each run one layer's fwd + bwd-weights + bwd-data "
                                   f"on a {SAMPLE_TOKENS}-token slice of the cfg5 step (layers round-robin), "
                                   f"oracle/tpp_oracle.py (the reference's per-element order); "
                                   f"{args.steps} steps after {n_warm} warm-up step(s)"},
        "e2e": {"value": round(val, 8), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# multi-rank plumbing without a GPU (gloo on CPU)
# ---------------------------------------------------------------------------

def run_dry(args, rank, world):
    """The launch / rank / timing logic of the N-rank bench on CPU: each rank
    runs a stand-in step (a 256^3 matmul per layer bucket + the GradSync
    exchange of scaled-down dW buckets), K timed steps between barriers, max
    over ranks, one JSON line from rank 0."""
    import torch
    import torch.distributed as dist

    from paper_2104_05755_b200 import parallel
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("gloo")
    sync = parallel.GradSync()
    a = torch.randn(256, 256)
    grads = [torch.zeros(DIMS[l] * DIMS[l + 1] // 1024) for l in range(len(DIMS) - 1)]
    flops_step = 2 * 256 ** 3 * len(grads) * world

    def step():
        for l in range(len(grads) - 1, -1, -1):
            grads[l].fill_(float(rank + 1))
            (a @ a).sum()
            sync.grad_ready(grads[l])
            sync.update_ready(lambda: None)
        sync.finish()

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(3):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        ms = (time.perf_counter() - t0) * 1e3
        if world > 1:
            t = torch.tensor([ms])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        times.append(ms)
    ok = all(float(g[0]) == float(sum(range(1, world + 1))) for g in grads)
    if rank == 0:
        ms_step = statistics.median(times) / args.steps
        print(json.dumps({
            "metric": METRIC, "value": round(flops_step / (ms_step * 1e-3) / 1e12, 6),
            "unit": "TFLOP/s (CPU stand-in)", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic", "config": bench_config(world),
            "dry_run": True, "allreduce_ok": ok, "backend": dist.get_backend() if world > 1 else None}),
            flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(n: int) -> int:
    """Re-launch this script as n ranks (one process per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time eager steps at N = 1 too")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--grad-dtype", choices=["fp32", "bf16"], default=None)
    ap.add_argument("--dry-run", action="store_true", help="CPU (gloo) run of the multi-rank plumbing")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if not args.dry_run and args.impl == "ours":
            import torch
            have = torch.cuda.device_count()
            if have < args.gpus and os.environ.get("TPP_BENCH_ONE_GPU") != "1":
                print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but {have} visible GPUs",
                                  "n_gpus": args.gpus}), flush=True)
                sys.exit(2)
        sys.exit(_spawn(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.dry_run:
        run_dry(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TPP_BENCH_BACKEND=gloo + TPP_BENCH_ONE_GPU=1: every rank on cuda:0 over
    # gloo -- a functional check of the N-rank path on a single-GPU box (not
    # a measurement: the ranks share one GPU)
    one_gpu = os.environ.get("TPP_BENCH_ONE_GPU") == "1"
    torch.cuda.set_device(0 if one_gpu else local)
    dist = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/tpp_nccl.%h.%p.log")
        import torch.distributed as dist_mod

        from paper_2104_05755_b200 import parallel
        parallel.init_from_env(os.environ.get("TPP_BENCH_BACKEND", "nccl"))
        dist = dist_mod
    run_ours(args, rank, world, dist)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
