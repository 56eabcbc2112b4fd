"""Print an ncu launch list (gpu__time_duration per launch) grouped by kernel."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        name = r[ki].split('(')[0].replace('void ', '').replace('dm::<unnamed>::', '')
        agg.setdefault(name, []).append(float(r[vi].replace(',', '')) / 1e3)
for k, v in agg.items():
    print(f"{k[:60]:60s} n={len(v):3d} mean={sum(v)/len(v):9.2f} us  min={min(v):9.2f}")
