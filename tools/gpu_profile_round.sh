# profile refresh: launch list of one bench step + ncu --set full of every launch of one step.
# Summaries are produced on the box (the .ncu-rep stays there: gpurun returns <= 64 MiB).
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_bench.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --launch-skip 150 --launch-count 50 -o /tmp/full_step -f python tools/launch_times.py > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
ncu -i /tmp/full_step.ncu-rep --page raw --csv > gpurun_out/full_step_raw.csv 2>/dev/null
python tools/ncu_summary.py full /tmp/full_step.ncu-rep gpurun_out/full_step.md --json gpurun_out/ncu_summary.json > /dev/null 2>&1; echo "summary rc=$?"
