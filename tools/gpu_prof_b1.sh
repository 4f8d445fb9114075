# Batch-1 launch list + ncu full (source) of the DMMA local kernel at batch 32 (n=2049).
mkdir -p gpurun_out
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 1"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M_b1.csv $CMD > gpurun_out/ncu_b1.log 2>&1; echo ncu=$?
CMD32="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_fdm_dmma -s 1 -c 1 -o gpurun_out/dmma_b32 $CMD32 > gpurun_out/ncu_dmma.log 2>&1; echo ncu2=$?
