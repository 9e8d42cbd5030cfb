bash tools/gpu_profile_round.sh
bash tools/gpu_workloads.sh
timeout 900 python bench.py > gpurun_out/bench_cifar.json 2> gpurun_out/bench_cifar.err; echo "cifar rc=$?"
timeout 900 python bench.py --weights trained --no-cpu > gpurun_out/bench_trained.json 2> gpurun_out/bench_trained.err; echo "trained rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
