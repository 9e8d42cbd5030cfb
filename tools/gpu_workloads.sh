# the other BASELINE configs and model files as bench lines (device + e2e), no CPU leg
for w in in64 1080p 1080p32; do
  timeout 900 python bench.py --workload $w --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
done
for m in trained sharp; do
  timeout 900 python bench.py --weights $m --no-cpu --headline-only > gpurun_out/bench_$m.json 2> gpurun_out/bench_$m.err; echo "$m rc=$?"
done
