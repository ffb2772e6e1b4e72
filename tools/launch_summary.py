"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel (dev helper)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
hdr = rows[hi]; data = rows[hi + 1:]
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
agg = collections.defaultdict(list)
for r in data:
    if len(r) <= vi or r[hdr.index('Metric Name')] != 'gpu__time_duration.sum':
        continue
    v = float(r[vi].replace(',', '')) * {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1, 'us': 1, 'msecond': 1e3, 'ms': 1e3}.get(r[ui], 1)
    agg[r[ki].split('(')[0][:60]].append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):5d} launches {sum(v):10.1f} us {100*sum(v)/tot:5.1f}%  mean {sum(v)/len(v):8.2f} us  {k}")
print(f"total {tot:.1f} us")
