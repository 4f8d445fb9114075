# Full ncu capture of the folded DMMA local kernel at config 5 (batch 32), plus a raw-metric dump.
mkdir -p gpurun_out
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32"
$CMD > gpurun_out/plain_local.log 2>&1; echo plain=$?
ncu --set full --clock-control none --import-source on -k regex:local_fdm_dmma -s 1 -c 1 -o gpurun_out/local_dmma $CMD > gpurun_out/ncu_local.log 2>&1; echo ncu=$?
ncu -i gpurun_out/local_dmma.ncu-rep --page raw --csv > gpurun_out/local_dmma_raw.csv 2>&1; echo raw=$?
ncu -i gpurun_out/local_dmma.ncu-rep --page details --csv > gpurun_out/local_dmma_details.csv 2>&1; echo det=$?
