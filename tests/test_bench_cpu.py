"""bench.py contract paths that need no GPU: the N-rank launch / timing
plumbing (``--gpus 2 --dry-run``: torch.distributed.run spawn, gloo, max over
ranks, one JSON line from rank 0) and the reference arm (``--impl reference``,
the oracle port on the host cores)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out: str):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


def test_bench_gpus2_dry_run_spawns_two_ranks():
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["dry_run"] and d["allreduce_ok"] and d["backend"] == "gloo"
    assert d["config"]["per_gpu_tokens"] == 4096 and d["steps"] == 2


def test_bench_reference_arm_one_step():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    # same config dict as the GPU arm at N = 1
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == json.loads(json.dumps(bench.bench_config(1)))
