# fused-block check: new parity test, full gpu suite, bench, per-launch times
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_codec.py -x -q -k "fused_encoder or trunk_kernel or pair_head" > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/memcheck.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 python tools/launch_times.py > gpurun_out/launch_times.txt 2>&1; head -20 gpurun_out/launch_times.txt
