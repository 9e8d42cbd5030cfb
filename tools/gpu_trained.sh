# GPU parity (whole -m gpu suite) + bench with random and trained weights
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest.log
for wt in random trained; do
  timeout 600 python bench.py --no-cpu --weights $wt > gpurun_out/bench_$wt.json 2> gpurun_out/bench_$wt.err; echo "bench $wt rc=$?"; cat gpurun_out/bench_$wt.json; tail -3 gpurun_out/bench_$wt.err
done
