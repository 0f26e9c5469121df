"""Summarize an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:60]:60s} {v[0]:6d} {v[1]:10.3f} ms {100 * v[1] / tot:5.1f}%")
print(f"total {tot:.3f} ms")
