"""Instruction mix (warp-level executed) by opcode from an ncu source csv."""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
c = Counter()
tot = 0
for r in rows[2:]:
    try:
        n = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    src = r[ix["Source"]].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", src)
    if not m:
        continue
    op = m.group(2)
    c[op] += n
    tot += n
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
print("total warp instr", tot, " per unit", tot / div)
for op, n in c.most_common(40):
    print(f"{op:12s} {n:14d} {n / tot * 100:6.2f}%  per-unit {n / div:8.3f}")
