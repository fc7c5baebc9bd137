"""Summarise an ncu --metrics gpu__time_duration.sum launch list CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]
ki, mi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
agg = collections.OrderedDict()
tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    v = float(r[mi].replace(',', ''))
    v = v / 1000 if r[ui] == 'ns' else (v * 1000 if r[ui] == 'ms' else v)
    name = r[ki].split('(')[0].replace('void ', '').replace('(anonymous namespace)::', '')[:70]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
    tot += v
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
print(f"total {tot:.1f} us over {sum(a[0] for a in agg.values())} launches; per step {tot / steps:.1f} us")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{t / steps:10.1f} us/step {100 * t / tot:5.1f}%  n/step={n / steps:6.1f}  avg={t / n:8.1f} us  {k}")
