"""Summarise an ncu --metrics gpu__time_duration.sum --csv log by kernel name."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = None
agg = defaultdict(lambda: [0, 0.0])
total = 0.0
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "nsecond")
        v = v / 1e6 if unit.startswith("n") else (v / 1e3 if unit.startswith("u") else v)
        agg[d["Kernel Name"][:70]][0] += 1
        agg[d["Kernel Name"][:70]][1] += v
        total += v
for n, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{v:10.3f} ms {100 * v / total:5.1f}% {c:5d}  {n}")
print(f"{total:10.3f} ms total")
