mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -k "operators or batched or zero or dimension or csr" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python tools/profile_ops.py --gmres 30 > gpurun_out/ops.log 2>&1; echo ops=$?
CMD="python tools/profile_ops.py --gmres 0 --only 'coarse solve' --reps 1 --batches 1,32"
eval $CMD > gpurun_out/plain.log 2>&1 && eval ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_coarse.csv $CMD > gpurun_out/ncu.log 2>&1; echo rc=$?
