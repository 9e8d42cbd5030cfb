# compute-sanitizer memcheck over the GPU suite (the reference-suite subprocess excluded)
mkdir -p gpurun_out
timeout 3000 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --target-processes all \
  python -m pytest tests/test_gpu_codec.py -m gpu -x -q > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"
tail -4 gpurun_out/memcheck.log
