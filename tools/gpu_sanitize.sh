# whole GPU suite under compute-sanitizer memcheck (+ synccheck on the fused-kernel tests)
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -x -q > gpurun_out/memcheck_all.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/memcheck_all.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_codec.py -x -q -k "fused_encoder or trunk_kernel" > gpurun_out/synccheck.log 2>&1; echo "synccheck rc=$?"; tail -4 gpurun_out/synccheck.log
