"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): per kernel count, total, mean."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; tot = collections.Counter(); cnt = collections.Counter()
for r in rows:
    if len(r) > 5 and r[0] == 'ID':
        hdr = {h: i for i, h in enumerate(r)}; continue
    if not hdr or len(r) <= 5 or r[hdr['Metric Name']] != 'gpu__time_duration.sum':
        continue
    k = r[hdr['Kernel Name']].split('(')[0].replace('void ', '')
    v = float(r[hdr['Metric Value']].replace(',', ''))
    u = r[hdr['Metric Unit']]
    v = v * {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3, 'second': 1e6}.get(u, 1e-3)   # -> us (ncu default ns)
    tot[k] += v; cnt[k] += 1
T = sum(tot.values())
print(f"total {T/1000:.3f} ms over {sum(cnt.values())} launches")
for k, v in tot.most_common():
    print(f"  {k[:64]:64s} n={cnt[k]:4d}  {v/1000:8.3f} ms  mean {v/cnt[k]:9.1f} us  {v/T*100:5.1f}%")
