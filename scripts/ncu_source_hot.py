"""Hottest SASS instructions of an ncu source page (csv from
`ncu -i R --page source --csv --print-source sass`), with stall split."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = []
for r in rows[2:]:
    try:
        n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    st = {k: int(r[ix[k]] or 0) for k in stalls}
    data.append((n, r[ix["Address"]], r[ix["Source"]], st, int(r[ix["Instructions Executed"]] or 0)))
tot = sum(d[0] for d in data)
print("total samples", tot)
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else None
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else None
if lo is not None:
    sel = [d for d in data if lo <= int(d[1], 16) < hi]
    print("range samples", sum(d[0] for d in sel), "frac", sum(d[0] for d in sel) / tot)
    agg = {}
    for d in sel:
        for k, v in d[3].items():
            agg[k] = agg.get(k, 0) + v
    print(sorted(agg.items(), key=lambda x: -x[1])[:8])
    for d in sel:
        top = sorted(d[3].items(), key=lambda x: -x[1])[:3]
        print(f"{d[1]:>6} {d[0]:7d} {d[4]:9d} {d[2][:60]:60s} {top}")
else:
    for d in sorted(data, key=lambda x: -x[0])[:40]:
        top = sorted(d[3].items(), key=lambda x: -x[1])[:3]
        print(f"{d[1]:>6} {d[0]:7d} {d[4]:9d} {d[2][:60]:60s} {top}")
