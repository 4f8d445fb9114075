mkdir -p gpurun_out
python tools/profile_ops.py --gmres 0 --only "local sum" --reps 1 --batches 32 > gpurun_out/plain.log 2>&1 && ncu --set full --import-source on -k regex:local_fdm_fold -s 1 -c 1 -o gpurun_out/fold python tools/profile_ops.py --gmres 0 --only "local sum" --reps 1 --batches 32 > gpurun_out/ncu2.log 2>&1; echo ncu=$?
