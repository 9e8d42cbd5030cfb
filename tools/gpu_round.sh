# round-end refresh: profiles, the other workloads, the default bench line and the reference arm
bash tools/gpu_profile_round.sh
bash tools/gpu_workloads.sh
timeout 900 python bench.py > gpurun_out/bench_cifar.json 2> gpurun_out/bench_cifar.err; echo "cifar rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
