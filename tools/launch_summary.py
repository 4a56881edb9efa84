"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel.
usage: python tools/launch_summary.py gpurun_out/launches.csv > profiles/x.txt"""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, rows = rows[0], rows[1:]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
if "Metric Name" in h:                       # lists with several metrics: the durations only
    im = h.index("Metric Name")
    rows = [r for r in rows if r[im] == "gpu__time_duration.sum"]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    ms = float(r[iv].replace(",", "")) * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(r[iu], 1e-6)
    name = r[ik].split("(")[0].strip()
    agg[name][0] += 1
    agg[name][1] += ms
tot = sum(a[1] for a in agg.values())
print(f"# {sys.argv[1]}: {len(rows)} launches, {tot:.3f} ms total (ncu: cold cache, serialised)")
print(f"{'ms':>10} {'share':>6} {'launches':>8}  kernel")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.3f} {100 * t / tot:5.1f}% {c:8d}  {k}")
