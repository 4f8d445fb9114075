# ncu --set full of the three top kernels of one SHS2 apply (config 5, batch 32)
mkdir -p gpurun_out
python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32 > gpurun_out/plain.log 2>&1; echo plain=$?
for k in local_fdm_dmma band_solve prolong_deflate xform_fft local_fdm_fast; do
  ncu --set full --clock-control none --import-source on -k "regex:$k" -s 1 -c 1 -o gpurun_out/k_$k python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32 > gpurun_out/ncu_$k.log 2>&1; echo $k=$?
done
