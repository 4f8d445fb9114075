# ncu --set full of selected kernels at config 5 (batch 32), one launch each; summaries via tools/ncu_brief.py
mkdir -p gpurun_out
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32"
$CMD > gpurun_out/plain_k.log 2>&1; echo plain=$?
for K in xform_fft combine_kernel band_solve_kernel prolong_deflate; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 0 -c 1 -o gpurun_out/k_$K $CMD > gpurun_out/ncu_$K.log 2>&1; echo $K=$?
done
