# Strip compensation variants: cfg4a count on both band paths + batch-1 coarse time; FFT timings.
mkdir -p gpurun_out
for c in 0 1 2 3; do
  echo "comp $c: $(HELM_STRIP_COMP=$c timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve' --batches 1 2>&1 | grep 'B=')"
  HELM_STRIP_COMP=$c timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
  HELM_STRIP_COMP=$c HELM_BAND_SEG_MAX=0 timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
done
timeout 300 python tools/profile_ops.py --gmres 0 --batches 1,32 2>&1 | grep "B="
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_M_b32.csv $CMD > gpurun_out/ncu_b32.log 2>&1; echo ncu=$?
