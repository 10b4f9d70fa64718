"""Summarise an ncu --csv launch list: per-kernel count, mean time, DRAM bytes, share of the step."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
hdr = rows[hi]
ki, vi, mi, idi = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name'), hdr.index('ID')
uni = hdr.index('Metric Unit')
per = collections.defaultdict(dict)
names = {}
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3,
         'byte': 1.0, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    per[r[idi]][r[mi]] = float(r[vi].replace(',', '')) * scale.get(r[uni], 1.0)
    names[r[idi]] = r[ki].split('(')[0].replace('void ', '').replace('<unnamed>::', '')
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get('gpu__time_duration.sum', 0)
    a[2] += m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)
tot = sum(a[1] for a in agg.values())
print(f"{'share':>7} {'launches':>8} {'mean_us':>9} {'MB/launch':>10} {'GB/s':>7}  kernel")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 16]:
    print(f"{t / tot * 100:6.2f}% {n:8d} {t / n:9.1f} {b / n / 1e6:10.1f} {b / n / (t / n * 1e-6) / 1e9 if t else 0:7.0f}  {k[:70]}")
print(f"total device time {tot / 1000:.1f} ms over {sum(a[0] for a in agg.values())} launches")
