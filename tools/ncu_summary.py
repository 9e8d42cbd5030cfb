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


RAW = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe (TC) % active"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor math % active"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem operand reads (TC) % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def full(path, out, js=None):
    """One row per profiled launch (raw page), with dram bytes per launch."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units = rr[0], rr[1]
    cols = {k: i for i, k in enumerate(hdr)}
    lines = ["| id | kernel | " + " | ".join(lab for _, lab in RAW) + " | dram bytes (r+w) |",
             "|---|---|" + "---:|" * (len(RAW) + 1)]
    dram = collections.defaultdict(list)
    for r in rr[2:]:
        name = kname(r[cols["Kernel Name"]])
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if m in cols:
                b += float(r[cols[m]].replace(",", "") or 0) * SCALE.get(units[cols[m]], 1)
        dram[name.split("<")[0]].append(b)
        vals = []
        for m, _ in RAW:
            if m in cols:
                v, u = r[cols[m]], units[cols[m]]
                vals.append(f"{v} {u}".strip() if u not in ("%", "") else v)
            else:
                vals.append("")
        lines.append(f"| {r[cols['ID']]} | `{name}` | " + " | ".join(vals) + f" | {b:.3e} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if js:
        try:
            cur = json.load(open(js))
        except (OSError, ValueError):
            cur = {}
        cur["dram_bytes_per_launch"] = {k: sum(v) / len(v) for k, v in dram.items()}
        cur["source"] = path
        json.dump(cur, open(js, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[5] if len(sys.argv) > 5 else None)
