mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python tools/profile_ops.py --batches 1,32 --gmres 0 > gpurun_out/ops.log 2>&1; echo ops=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M.csv python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32 > gpurun_out/ncu.log 2>&1; echo ncu=$?
