"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
h = rows[hi]; data = rows[hi + 1:]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0]); tot = 0
for r in data:
    if len(r) <= vi: continue
    v = float(r[vi].replace(',', ''))
    v *= {'nsecond': 1, 'usecond': 1e3, 'msecond': 1e6}.get(r[ui], 1)
    name = r[ki].split('(')[0][:60]
    agg[name][0] += 1; agg[name][1] += v; tot += v
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t/1e6:9.3f} ms {100*t/tot:5.1f}% n={c:5d} avg={t/c/1e3:8.1f} us  {k}")
print(f"total {tot/1e6:.3f} ms over {sum(c for c,_ in agg.values())} launches")
