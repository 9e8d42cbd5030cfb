mkdir -p gpurun_out
timeout 1500 python tests/golden/make_sharp.py gpurun_out/sharp.pilw 2>&1 | tail -12
timeout 600 python tools/sharp_eval.py gpurun_out/sharp.pilw 1024
timeout 600 python tools/sharp_eval.py tests/golden/trained.pilw 1024
