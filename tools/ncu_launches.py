"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel launches, total device time and share (cold-cache, serialised)."""
import csv, re, sys
from collections import OrderedDict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr, rows = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = OrderedDict()
for r in rows:
    name = re.sub(r"\(.*", "", r[ki]).replace("<unnamed>::", "").replace("void ", "")
    t = float(r[vi]) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}[r[ui]]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += t
tot = sum(v[1] for v in agg.values())
print(f"| kernel | launches | total us | share |\n|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
print(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.1f} | 100% |")
