"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel count / mean µs, in launch order."""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = OrderedDict()
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') != 'gpu__time_duration.sum':
            continue
        name = d['Kernel Name'].split('(')[0][:70] + ' ' + d.get('Grid Size', '')
        v = float(d['Metric Value'].replace(',', ''))
        unit = d.get('Metric Unit', 'ns')
        us = v / 1000 if unit in ('ns', 'nsecond') else (v if unit in ('us', 'usecond') else v * 1000)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
for k, (n, t) in agg.items():
    print(f"{n:4d} x {t / n:9.2f} us  {k}")
