# band_seg chunk configs at batch 1 + launch list of one batch-1 M^-1 (n=2049).
mkdir -p gpurun_out
for c in 0 1 2 3; do
  echo "segcfg $c: $(HELM_SEG_CFG=$c timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve,M^-1' --batches 1 2>&1 | grep 'B=' | tr '\n' ' ')"
done
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 1"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M_b1.csv $CMD > gpurun_out/ncu_b1.log 2>&1; echo ncu=$?
