# ncu --set full of one launch of kernel $K (regex) from a bench-like step; summaries made on the box
K=${K:-tc3_block_kernel}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${NCU_SKIP:-1} -c 1 -o /tmp/one -f python tools/launch_times.py > gpurun_out/ncu_one.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/one.ncu-rep --page raw --csv > gpurun_out/one_raw.csv 2>/dev/null
ncu -i /tmp/one.ncu-rep --page source --csv --print-source sass > gpurun_out/one_src.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/one_src.csv 40 > gpurun_out/one_stalls.txt 2>&1
python tools/ncu_summary.py full /tmp/one.ncu-rep gpurun_out/one.md > /dev/null 2>&1
cp /tmp/one.ncu-rep gpurun_out/one.ncu-rep
ls -la gpurun_out/one*
