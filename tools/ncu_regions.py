"""Stall samples of an ncu source page (SASS) aggregated over address windows, by stall reason.

    ncu -i rep --page source --csv --print-source sass > src.csv; python tools/ncu_regions.py src.csv [window]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
W = int(sys.argv[2]) if len(sys.argv) > 2 else 64
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[iS] or 0) for r in data) or 1.0
for k in range(0, len(data), W):
    seg = data[k:k + W]
    s = sum(float(r[iS] or 0) for r in seg)
    if s / tot < 0.005:
        continue
    rs = collections.Counter()
    for r in seg:
        for c in reasons:
            rs[c] += float(r[h.index(c)] or 0)
    ops = collections.Counter((r[1].split()[1] if r[1].strip().startswith("@") else r[1].split()[0]) for r in seg)
    ex = max(int(r[iE] or 0) for r in seg)
    top = ", ".join(f"{c[6:]} {v / tot * 100:.1f}" for c, v in rs.most_common(3))
    print(f"{k:5d} {s / tot * 100:5.1f}% ex~{ex:>7} [{top}] {dict(ops.most_common(4))}")
