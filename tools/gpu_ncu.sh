# ncu --set full captures of selected kernels (one launch each) from one bench-like step
K=${NCU_KERNELS:-"tc3_conv_kernel rans_decode_kernel"}
for k in $K; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s ${NCU_SKIP:-2} -c 1 -o gpurun_out/ncu_$k -f python tools/launch_times.py > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done
