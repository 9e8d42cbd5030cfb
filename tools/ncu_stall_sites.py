"""Stall samples of one kernel in an ncu report, attributed to the kernel's
own source lines (inlined helpers such as mbar_wait folded into their call
site): python tools/ncu_stall_sites.py report.ncu-rep [min_line]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
min_line = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hdr]
iS = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [(j, c) for j, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
seq, line = [], None
for r in rows[hdr + 1:]:
    if r and r[0].isdigit():
        line = int(r[0])
    elif r and r[0]:
        line = None
    elif len(r) > 3 and r[2].startswith("0x"):
        seq.append((int(r[2], 16), line, r[3], r))
seq.sort()
site, cur = {}, None
src = {}
for addr, ln, sass, r in seq:
    if ln is not None and ln >= min_line:
        cur = ln
    key = cur
    n = int(r[iS] or 0)
    d = site.setdefault(key, [0, {}])
    d[0] += n
    for j, c in stall_cols:
        v = int(r[j] or 0) if (r[j] or "0").isdigit() else 0
        if v:
            d[1][c] = d[1].get(c, 0) + v
tot = sum(v[0] for v in site.values())
print("total samples", tot)
for k, (n, st) in sorted(site.items(), key=lambda kv: -kv[1][0])[:30]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{n:7d} {100.0 * n / max(tot, 1):5.1f}%  line {k}  {top}")
