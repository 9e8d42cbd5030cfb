# profile refresh for the round: launch list of one headline bench step (ncu
# gpu__time_duration, cold-cache serialised), a --set full capture of every
# kernel of one fast step, and one exact-network conv launch. Summaries are
# produced on the box (.ncu-rep files stay there: gpurun returns <= 64 MiB).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --headline-only > gpurun_out/ncu_bench.log 2>&1; echo "launch list rc=$?"
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
python tools/ncu_summary.py launches gpurun_out/launches.csv gpurun_out/launches.md > /dev/null 2>&1; echo "launches md rc=$?"
# one exact-network block conv (the exact step's dominant kernel)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_kernel -s 8 -c 1 -o /tmp/exact_conv -f python tools/launch_times.py 32 2048 exact > /dev/null 2>&1; echo "exact conv rc=$?"
python tools/ncu_summary.py full /tmp/exact_conv.ncu-rep gpurun_out/exact_conv.md > /dev/null 2>&1; echo "exact md rc=$?"
timeout 1500 python bench.py --workload coder > gpurun_out/bench_coder.json 2> gpurun_out/bench_coder.err; echo "coder rc=$?"
