timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve,M^-1' --batches 8,32 2>&1 | grep "B="
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:strip_reduce_kernel --csv --log-file gpurun_out/sr.csv $CMD > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/sr.csv
