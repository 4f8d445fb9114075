# ncu full captures of the compensated strip kernels at batch 1 (n=2049).
mkdir -p gpurun_out
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 1"
$CMD > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:strip_reduce_c -s 1 -c 1 -o gpurun_out/sred_b1 $CMD > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:strip_left_fused -s 1 -c 1 -o gpurun_out/sleft_b1 $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_seg_kernel -s 1 -c 1 -o gpurun_out/seg44_b1 $CMD > gpurun_out/ncu3.log 2>&1; echo ncu3=$?
