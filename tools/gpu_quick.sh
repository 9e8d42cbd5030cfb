# quick GPU check: parity tests + bench (no CPU leg) + live per-launch times
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest.log
timeout 600 python bench.py --no-cpu ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 300 python tools/launch_times.py > gpurun_out/launch_times.txt 2>&1; tail -50 gpurun_out/launch_times.txt
