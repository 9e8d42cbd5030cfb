mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "lane or rans or coder or static or round_trip" > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest.log
timeout 1200 python bench.py --workload coder > gpurun_out/bench_coder.json 2> gpurun_out/bench_coder.err; echo "coder rc=$?"; cat gpurun_out/bench_coder.json; tail -3 gpurun_out/bench_coder.err
