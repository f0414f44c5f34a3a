"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv, sys
from collections import defaultdict
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.DictReader(lines))
d = defaultdict(list)
for r in rows:
    if r['Metric Name'] == 'gpu__time_duration.sum':
        scale = {'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3}.get(r['Metric Unit'], 1e-3)
        d[r['Kernel Name'].split('(')[0]].append(float(r['Metric Value'].replace(',', '')) * scale)
tot = sum(sum(v) for v in d.values())
for k, v in d.items():
    v = sorted(v)
    print(f"{k:40s} n={len(v):4d} median_us={v[len(v)//2]:9.2f} min={v[0]:9.2f} max={v[-1]:9.2f} share={sum(v)/tot:6.1%}")
