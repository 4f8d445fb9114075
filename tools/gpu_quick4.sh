# GPU tests + op timings + fixed GMRES + cfg4a count + batch-32 launch list.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_ops.py --gmres 0 --batches 1,32 2>&1 | grep "B="
timeout 300 python tools/gmres_fixed.py 50 2>&1 | tail -1
timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_M_b32.csv $CMD > gpurun_out/ncu_b32.log 2>&1; echo ncu=$?
