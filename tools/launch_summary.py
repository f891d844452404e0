#!/usr/bin/env python
"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
    python tools/launch_summary.py gpurun_out/X_launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
agg = collections.OrderedDict()
for r in rows[1:]:
    a = agg.setdefault(r[ki][:70], [0, 0.0])
    a[0] += 1
    a[1] += float(r[vi].replace(',', ''))
tot = sum(t for n, t in agg.values() if 'k_peak' not in '')
for k, (n, t) in agg.items():
    print(f"{n:6d} {t / 1e6:10.3f} ms {t / n / 1e3:10.1f} us/launch  {k}")
