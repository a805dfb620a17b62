"""Summarise an ncu launch-list csv (gpu__time_duration per launch): time share per kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; L = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d['Metric Name'] == 'gpu__time_duration.sum':
            v = float(d['Metric Value'].replace(',', ''))
            v = v / 1e3 if d['Metric Unit'] == 'ns' else (v * 1e3 if d['Metric Unit'] == 'ms' else v)
            L.append((d['Kernel Name'].split('(')[0].replace('void ', ''), v))
agg = collections.defaultdict(lambda: [0, 0.0])
for k, t in L: agg[k][0] += 1; agg[k][1] += t
tot = sum(v[1] for v in agg.values())
print(f"{len(L)} launches, {tot:.1f} us total")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:72]:72s} {n:4d} {t:9.1f} us {100*t/tot:5.1f}%  ({t/n:7.1f} us/launch)")
