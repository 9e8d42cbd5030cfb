"""Stall breakdown of an ncu source-page CSV (--page source --csv --print-source sass):
totals per stall reason and the top instructions with their dominant reasons."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[1], rows[2:]
reasons = [c for c in h if c.startswith('stall_') and '(Not' not in c]
ix = {c: h.index(c) for c in reasons}
isrc, iall = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = {c: sum(int(r[ix[c]] or 0) for r in data) for c in reasons}
T = sum(tot.values())
print("total", T)
for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]:
    print(f"  {c:24s} {v:7d} {100*v/max(T,1):5.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for k, r in enumerate(sorted(range(len(data)), key=lambda i: -int(data[i][iall] or 0))[:n]):
    d = data[r]
    top = sorted(((int(d[ix[c]] or 0), c) for c in reasons), reverse=True)[:2]
    print(f"{r:5d} {int(d[iall] or 0):6d} {d[isrc][:70]:70s} {top}")
