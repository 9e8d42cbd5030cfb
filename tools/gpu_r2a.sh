# round-2 first check: microbench FFMA/FFMA2 rate, then the GPU suite as committed
mkdir -p gpurun_out
./tools/micro/ffma_rate > gpurun_out/ffma_rate.txt 2>&1; cat gpurun_out/ffma_rate.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -i "model name\|^CPU(s)" 
python -c "import numpy; numpy.show_config()" 2>&1 | grep -A3 -i "openblas config\|SIMD" | head
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest.log
