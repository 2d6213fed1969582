"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("(anonymous namespace)::", "")[:70]
    if len(sys.argv) > 2 and gi is not None:
        name += " grid=" + r[gi]
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"total {tot / 1e3:.3f} ms over {sum(c for c, _ in agg.values())} launches")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}% {c:6d} launches  avg {t / c:8.1f} us  {k}")
