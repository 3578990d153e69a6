"""Summarise an ncu launch list (gpu__time_duration.sum per launch) of
bench.py into per-step kernel shares: the library's kernels are grouped into
training steps (a step starts at each first forward GEMM after a split-SGD
or at the start), one representative step is printed with each launch's
duration and share, plus the per-class totals over all complete steps.
Usage: python tools/launch_share.py launches.csv > profiles/<name>.txt"""
import collections
import csv
import statistics
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
ki, ni, mi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
seq = []
for r in rows[hi + 1:]:
    if len(r) > mi and r[ni] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0].replace("void ", "")
        if "tpp::" in r[ki] or "tc::" in name or "brgemm" in name:
            seq.append((name, float(r[mi].replace(",", ""))))
# a step = 4 forward GEMMs, the softmax-CE kernel, then per layer (last first)
# backward-data + backward-weights (split-SGD fused at one rank): 12 launches
# anchored on the softmax_xent kernel
NB, NA = 4, 7
labels = ["fwd0", "fwd1", "fwd2", "fwd3", "xent", "dx3", "dw3", "dx2", "dw2", "dx1", "dw1", "dw0"]
steps = []
for k, (name, _) in enumerate(seq):
    if "softmax_xent" in name and k >= NB and k + NA < len(seq):
        steps.append(seq[k - NB:k + NA + 1])
print(f"# ncu launch list ({sys.argv[1]}): {len(seq)} library launches, {len(steps)} complete training steps")
print("# cold-cache, serialised per-launch times (ncu --metrics gpu__time_duration.sum --clock-control none):")
print("# compare SHARES with bench.py's live breakdown, not absolutes")
if steps:
    med = [statistics.median(s[i][1] for s in steps) for i in range(len(labels))]
    tot = sum(med)
    print(f"median step (sum of launches): {tot / 1e3:.1f} us")
    for lab, (name, _), v in zip(labels, steps[-1], med):
        print(f"  {lab:5s} {name[:48]:48s} {v / 1e3:8.1f} us  {100 * v / tot:5.1f} %")
    cls = collections.defaultdict(float)
    for (name, _), v in zip(steps[-1], med):
        cls[name] += v
    print("per kernel class:")
    for name, v in sorted(cls.items(), key=lambda t: -t[1]):
        print(f"  {name[:60]:60s} {v / 1e3:8.1f} us  {100 * v / tot:5.1f} %")
