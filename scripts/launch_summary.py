"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict

SCALE = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
         "s": 1e9, "second": 1e9}
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
data = [dict(zip(h, r)) for r in rows[hi + 1:] if len(r) == len(h)]
agg = defaultdict(lambda: [0, 0.0])
for d in data:
    k = d["Kernel Name"].split("(")[0][:64]
    v = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:n]:
    print(f"{k:64s} {c:5d} {t / 1e6:10.3f} ms {100 * t / tot:6.2f}%")
print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
