"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    agg.setdefault(r[ki].split('(')[0][:60], []).append(float(r[vi].replace(',', '')))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:62s} n={len(v):3d} total={sum(v)/1e6:9.3f} ms  mean={sum(v)/len(v)/1e6:8.3f} ms  share={sum(v)/tot:6.1%}")
