"""Summarise ncu reports / launch lists into profiles/ (text, committed)."""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_active.avg", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
]


def raw(rep, idx=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2 + idx]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def summarize(rep, title, idx=0):
    d = raw(rep, idx)
    lines = [f"# {title}", f"report: {rep}", f"kernel: {d.get('Kernel Name', ('?',))[0]}"]
    for k in KEYS:
        for name, (v, u) in d.items():
            if name == k or name.endswith("." + k):
                lines.append(f"{k:75s} {v} {u}")
                break
    return "\n".join(lines)


def launches(csv_path, out):
    rows = [r for r in csv.reader(l for l in open(csv_path) if not l.startswith("=="))]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = {}
    for r in rows[1:]:
        name = r[ki].split("(")[0][:80]
        v = float(r[vi].replace(",", ""))
        if r[ui] == "usecond":
            v *= 1000
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    lines = [f"# ncu launch list: {csv_path}", "# kernel | launches | total ns | share", ]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{n:80s} {c:6d} {t:14.0f} {t / tot:7.3f}")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "rep":
        print(summarize(sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 0))
    else:
        launches(sys.argv[2], sys.argv[3])
