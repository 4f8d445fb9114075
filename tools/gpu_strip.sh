mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python tools/profile_ops.py --gmres 0 --reps 5 > gpurun_out/ops.log 2>&1; echo ops=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M.csv python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32 > gpurun_out/ncu.log 2>&1; echo ncu=$?
