"""Dev tool: aggregate an ncu --csv gpu__time_duration launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, mi, vi, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
        continue
    v = float(r[vi].replace(',', ''))
    u = r[ui]
    v = v / 1e3 if u in ('nsecond', 'ns') else (v * 1e3 if u in ('msecond', 'ms') else v)
    a = agg.setdefault(r[ki][:90], [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for k, v in agg.items() if 'probe' not in k)
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    if 'probe' in k:
        continue
    print(f"{v / tot * 100:6.2f}% {c:5d} {v / c:10.1f}us/launch {v / steps:10.1f}us/step  {k}")
print(f"total {tot / steps:.1f} us/step")
