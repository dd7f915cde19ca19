"""Opcode mix of an ncu source-page export (--page source --csv --print-source sass):
   python scripts/sass_mix.py gpurun_out/prof_X_src.csv [pixels]   (warp instructions executed per opcode)"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
si, ei = h.index("Source"), h.index("Instructions Executed")
mix = collections.Counter()
tot = 0
for r in rows[hi + 1:]:
    try:
        n = int(r[ei])
    except (ValueError, IndexError):
        continue
    op = r[si].split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    mix[o.split(".")[0]] += n
    tot += n
px = float(sys.argv[2]) if len(sys.argv) > 2 else None
for o, n in mix.most_common(30):
    print(f"{o:12s} {n:14d} {100.0 * n / tot:5.1f}%" + (f"  {32.0 * n / px:6.2f}/px" if px else ""))
print("total", tot, f"{32.0 * tot / px:.1f}/px" if px else "")
