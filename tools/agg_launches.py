import csv, collections, sys
path = sys.argv[1]; last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
tail = data[-last:] if last else data
agg = collections.defaultdict(lambda: [0, 0.0])
for d in tail:
    name = d['Kernel Name'].split('(')[0][:70]
    v = float(d['Metric Value']); u = d['Metric Unit']
    v *= {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3, 's': 1e6, 'second': 1e6}.get(u, 1.0)
    agg[name][0] += 1; agg[name][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{k:70s} n={v[0]:5d} total={v[1]:10.1f}us share={v[1]/tot*100:5.1f}% avg={v[1]/v[0]:8.2f}us")
print('launches', len(tail), 'total device us', round(tot, 1))
