mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rans_decode -s 2 -c 1 -o gpurun_out/ncu_dec1k -f python tools/coder_probe.py 1024 22 > gpurun_out/ncu_dec1k.log 2>&1; echo rc=$?
ncu -i gpurun_out/ncu_dec1k.ncu-rep --page details --csv 2>/dev/null | grep -i "stall\|Warp Cycles\|Issued\|Eligible\|Registers\|Block Size\|Grid Size\|Achieved Occ" | head -40
ncu -i gpurun_out/ncu_dec1k.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/dec1k_raw.csv
