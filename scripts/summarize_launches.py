"""Summarise an ncu --csv launch list: per kernel name, count and mean of each metric."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, ii, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
per = OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    per.setdefault((r[ii], r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
agg = OrderedDict()
for (i, name), m in per.items():
    short = name.split("(")[0][:40]
    a = agg.setdefault(short, {"n": 0})
    a["n"] += 1
    for k, v in m.items():
        a[k] = a.get(k, 0.0) + v
for name, a in agg.items():
    n = a.pop("n")
    print(f"{name:42s} n={n:3d} " + " ".join(f"{k.split('.')[0].split('__')[-1]}={v / n:.4g}" for k, v in a.items()))
