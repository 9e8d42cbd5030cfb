"""Summarise ncu output into profiles/.

    python tools/ncu_summary.py launches <launches.csv> <out.md>
    python tools/ncu_summary.py full <prof.ncu-rep> <out.md> [--json profiles/ncu_summary.json]

`launches`: per-kernel launch counts, device time and share of the step
from an `ncu --metrics gpu__time_duration.sum` launch list (cold-cache,
serialised: compare shares, not absolutes). `full`: key metrics of each
profiled launch of an `ncu --set full` capture, plus dram bytes per launch
(dram__bytes_read.sum + dram__bytes_write.sum) for bench.py's roofline.
"""
import collections
import csv
import io
import json
import subprocess
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}


def kname(s):
    s = s.replace("void ", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    return s.split("(")[0]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        us = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        agg[kname(r[ki])][0] += 1
        agg[kname(r[ki])][1] += us
    tot = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {us / 1e3:.3f} | {100 * us / tot:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Achieved Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Grid Size", "Block Size", "Executed Ipc Active", "Issue Slots Busy"]


def full(path, out, js=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    idx = {k: i for i, k in enumerate(h)}
    per = collections.OrderedDict()
    for r in rows[1:]:
        key = (r[idx["ID"]], kname(r[idx["Kernel Name"]]))
        if r[idx["Metric Name"]] in WANT:
            per.setdefault(key, {})[r[idx["Metric Name"]]] = f"{r[idx['Metric Value']]} {r[idx['Metric Unit']]}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units = rr[0], rr[1]
    cols = {k: i for i, k in enumerate(hdr)}
    dram = {}
    tensor = {}
    for r in rr[2:]:
        name = kname(r[cols["Kernel Name"]])
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if m in cols:
                v = float(r[cols[m]].replace(",", "") or 0)
                u = units[cols[m]]
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                b += v
        dram.setdefault(name, []).append(b)
        for m in cols:
            if m.startswith("sm__pipe_tensor") and "pct_of_peak_sustained_active" in m:
                tensor.setdefault(name, {})[m] = r[cols[m]]
    lines = []
    for (i, k), d in per.items():
        lines.append(f"### launch {i}: `{k}`")
        for m in WANT:
            if m in d:
                lines.append(f"- {m}: {d[m]}")
        if k in dram:
            lines.append(f"- dram bytes (read+write): {dram[k][0]:.0f}")
        for m, v in tensor.get(k, {}).items():
            lines.append(f"- {m}: {v}")
        lines.append("")
    open(out, "w").write("\n".join(lines))
    print("\n".join(lines))
    if js:
        try:
            cur = json.load(open(js))
        except OSError:
            cur = {}
        cur.setdefault("dram_bytes_per_launch", {})
        for k, v in dram.items():
            base = k.split("<")[0]
            cur["dram_bytes_per_launch"][base] = sum(v) / len(v)
        json.dump(cur, open(js, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[5] if len(sys.argv) > 5 else None)
