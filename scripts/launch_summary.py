"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel (dev tool).

    python scripts/launch_summary.py launches.csv "header line" > profiles/<name>.txt"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi or not r[vi]:
        continue
    name = re.sub(r"^(void )?<unnamed>::", "", r[ki]).split("(")[0]
    name = name.replace("<(bool)0>", "<0>").replace("<(bool)1>", "<1>").replace("<false>", "<0>").replace("<true>", "<1>")
    us = float(r[vi].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
    n, t = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, t + us)
total = sum(t for _, t in agg.values())
print(sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
print(f"{'kernel':40s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:40s} {n:8d} {t:10.1f} {t / n:9.2f} {t / total:6.3f}")
