# the other BASELINE configs as bench lines (device + e2e), no CPU leg
for w in in64 1080p coder; do
  timeout 900 python bench.py --workload $w --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
done
