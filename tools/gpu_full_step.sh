mkdir -p gpurun_out
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
starts = [n for n, (_, k) in enumerate(ids) if "twar_forward" in k]
print(starts[-1], len(ids) - starts[-1])
PY
)
echo "full capture: skip $SKIP count $COUNT"
timeout 1500 ncu --set full --clock-control none --launch-skip $SKIP --launch-count $COUNT -o /tmp/full_step -f python tools/launch_times.py > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
python tools/ncu_summary.py full /tmp/full_step.ncu-rep gpurun_out/full_step.md --json gpurun_out/ncu_summary.json > /dev/null 2>&1; echo "summary rc=$?"
