# compute-sanitizer memcheck over the GPU suite's exact-network, coder and multi-device tests
mkdir -p gpurun_out
timeout 3000 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --target-processes all \
  python -m pytest tests/test_gpu_codec.py -m gpu -x -q -k "exact or lane or round_trip or devices or sharp or static or vqvae" \
  > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/memcheck.log; grep -c "Invalid\|ERROR SUMMARY" gpurun_out/memcheck.log
