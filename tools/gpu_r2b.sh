# exact network: GPU suite + smoke + per-launch times of both numerics
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
timeout 300 python tools/launch_times.py 32 8192 exact > gpurun_out/lt_exact.txt 2>&1; tail -40 gpurun_out/lt_exact.txt
timeout 300 python tools/launch_times.py 32 8192 fast > gpurun_out/lt_fast.txt 2>&1; tail -8 gpurun_out/lt_fast.txt
