#!/usr/bin/env python
"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
k, v, u = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
for r in rows[hdr_i + 1:]:
    if len(r) <= v:
        continue
    name = r[k].split("(")[0][-60:]
    tot[name][0] += 1
    tot[name][1] += float(r[v].replace(",", "")) * scale.get(r[u], 1e-6)
allms = sum(t[1] for t in tot.values())
for name, (n, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{ms:10.3f} ms {100 * ms / allms:5.1f}% {n:6d}x  {name}")
print(f"{allms:10.3f} ms total")
