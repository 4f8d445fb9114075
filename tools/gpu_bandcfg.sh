# A/B of band-solve launch configurations at batch 32 (coarse solve, n=2049).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
for c in 0 1 2 3 4 5 6; do
  echo "cfg $c: $(HELM_BAND_CFG=$c timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve' --batches 32 2>&1 | grep -i 'coarse solve' | tail -1)"
done
echo "seg: $(HELM_BAND_SEG_MAX=64 timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve' --batches 32 2>&1 | grep -i 'coarse solve' | tail -1)"
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 1"
$CMD > gpurun_out/plain_b1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xform_fft -s 1 -c 1 -o gpurun_out/fft_b1 $CMD > gpurun_out/ncu_fft.log 2>&1; echo ncu_fft=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_seg_kernel -s 1 -c 1 -o gpurun_out/seg_b1 $CMD > gpurun_out/ncu_seg.log 2>&1; echo ncu_seg=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:strip_left_fused -s 1 -c 1 -o gpurun_out/stripl_b1 $CMD > gpurun_out/ncu_sl.log 2>&1; echo ncu_sl=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_fdm_fast -s 1 -c 1 -o gpurun_out/fast_b1 $CMD > gpurun_out/ncu_fast.log 2>&1; echo ncu_fast=$?
