# profile refresh: launch list of one bench step + ncu --set full of every launch of one step.
# Summaries are produced on the box (the .ncu-rep stays there: gpurun returns <= 64 MiB).
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_bench.log 2>&1; echo "launch list rc=$?"
# launch list of tools/launch_times.py (3 warm-up steps + 1): the full capture covers the last step
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/lt_launches.csv python tools/launch_times.py > /dev/null 2>&1
read SKIP COUNT < <(python - <<'PY'
import csv
rows = list(csv.reader(open("/tmp/lt_launches.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
ki, ii = rows[hi].index("Kernel Name"), rows[hi].index("ID")
ids = []
for r in rows[hi + 1:]:
    if len(r) > ki and (not ids or ids[-1][0] != r[ii]):
        ids.append((r[ii], r[ki]))
starts = [n for n, (_, k) in enumerate(ids) if "twar_forward_kernel" in k]
print(starts[-1], len(ids) - starts[-1])
PY
)
echo "full capture: skip $SKIP count $COUNT"
timeout 1500 ncu --set full --clock-control none --launch-skip $SKIP --launch-count $COUNT -o /tmp/full_step -f python tools/launch_times.py > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
ncu -i /tmp/full_step.ncu-rep --page raw --csv > gpurun_out/full_step_raw.csv 2>/dev/null
python tools/ncu_summary.py full /tmp/full_step.ncu-rep gpurun_out/full_step.md --json gpurun_out/ncu_summary.json > /dev/null 2>&1; echo "summary rc=$?"
python tools/ncu_summary.py launches gpurun_out/launches.csv gpurun_out/launches.md > /dev/null 2>&1; echo "launches md rc=$?"
