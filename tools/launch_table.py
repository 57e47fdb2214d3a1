"""Per-kernel duration table from an ncu --metrics gpu__time_duration.sum CSV log."""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i0]
kn, mv = h.index("Kernel Name"), h.index("Metric Value")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
seq = [(r[kn].split("(")[0][:70], float(r[mv].replace(",", ""))) for r in rows[i0 + 1:] if len(r) > mv]
seq = seq[skip:]
tot = OrderedDict()
for n, v in seq:
    a = tot.setdefault(n, [0, 0.0]); a[0] += 1; a[1] += v
for n, (c, v) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:72s} n={c:4d} total={v/1e3:9.1f} us  avg={v/c/1e3:8.1f} us")
