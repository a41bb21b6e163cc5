"""Per-kernel device time from an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
t, c = defaultdict(float), defaultdict(int)
for r in rows[start + 1:]:
    if len(r) < len(h):
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    n = r[ki].split("(")[0].split("::")[-1][:44]
    t[n] += v
    c[n] += 1
tot = sum(t.values())
for n, v in sorted(t.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{n:46s} {c[n]:4d} {v / 1e6:9.3f} ms {100 * v / tot:5.1f}%")
