"""Per-source-line warp-stall samples and executed instructions of an ncu report (cuda,sass view)."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
cur = None; agg = {}
for r in rows[3:]:
    if len(r) < 8: continue
    if r[0] != '':
        cur = (r[0], r[1][:100]); agg.setdefault(cur, [0, 0]); continue
    try:
        agg[cur][0] += int(r[4]); agg[cur][1] += int(r[7])
    except (ValueError, KeyError): pass
tot = sum(v[0] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v[0]*100/tot:5.1f}% {v[1]:>11d}  {k[0]:>5s} {k[1]}")
