mkdir -p gpurun_out
CMD="python tools/profile_ops.py --gmres 0 --only 'coarse solve' --reps 1 --batches 1,32"
eval $CMD > gpurun_out/plain.log 2>&1 && eval ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_coarse.csv $CMD > gpurun_out/ncu.log 2>&1; echo rc=$?
