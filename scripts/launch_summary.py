"""Summarise an ncu launch list (gpu__time_duration per launch) for the LAST build step."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[h]; body = rows[h + 1:]
ik, iv, iid = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('ID')
seq = [(int(r[iid]), r[ik], float(r[iv].replace(',', ''))) for r in body if len(r) == len(hdr)]

# split at occupancy kernel launches (first kernel of a build)
starts = [i for i, (_, k, _) in enumerate(seq) if 'k_occupancy' in k]
last = seq[starts[-1]:] if starts else seq
tot = sum(v for _, _, v in last)
agg = collections.OrderedDict()
for _, k, v in last:
    name = k.split('(')[0].replace('void ', '')[:48]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1; a[1] += v
print(f"last build: {len(last)} launches, {tot/1e3:.1f} us (ncu serialised)")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k:50s} n={c:4d} {v/1e3:9.1f} us  {v/tot*100:5.1f}%")
if '-v' in sys.argv:
    for _, k, v in last: print(f"    {k.split('(')[0][:60]:60s} {v/1e3:9.2f} us")
