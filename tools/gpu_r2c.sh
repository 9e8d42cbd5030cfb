mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "exact or vqvae or smoke or trained" > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest.log
timeout 300 python tools/launch_times.py 32 8192 exact > gpurun_out/lt_exact.txt 2>&1; cat gpurun_out/lt_exact.txt | sort -k2 -n -r | head -12; tail -1 gpurun_out/lt_exact.txt
