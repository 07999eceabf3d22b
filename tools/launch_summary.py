"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
hdr = rows[hi]; ik = hdr.index('Kernel Name'); iv = hdr.index('Metric Value'); iu = hdr.index('Metric Unit')
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= iv: continue
    v = float(r[iv].replace(',', '')); u = r[iu]
    ns = v * 1e3 if u == 'usecond' else (v * 1e6 if u == 'msecond' else v)
    name = r[ik].split('(')[0].replace('void ', '')
    agg[name][0] += 1; agg[name][1] += ns
tot = sum(v for _, v in agg.values())
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{100*v/tot:5.1f}% {v/1e6:10.3f} ms n={n:5d} {k[:90]}")
