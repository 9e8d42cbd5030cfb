mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_reference_suite.py -m gpu -x -q > gpurun_out/pytest_ref.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/pytest_ref.log; grep -E "passed|failed|error" gpurun_out/reference_suite.log | tail -5; grep -E "^FAILED|^ERROR" gpurun_out/reference_suite.log | head -40
