mkdir -p gpurun_out
python tools/profile_ops.py --gmres 0 --only "coarse solve" --reps 1 --batches 1 > gpurun_out/plain.log 2>&1 && ncu --set full --import-source on -k "regex:band_solve" -s 0 -c 1 -o gpurun_out/band1 python tools/profile_ops.py --gmres 0 --only "coarse solve" --reps 1 --batches 1 > gpurun_out/ncu.log 2>&1; echo ncu=$?
