# quick check + launch list of one M^-1 apply (config 5, batch 32)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not large" > gpurun_out/pytest_quick.log 2>&1; echo pytest=$?
timeout 600 python tools/profile_ops.py --gmres 0 --reps 5 --only "${1:-local sum,coarse solve,M^-1}" > gpurun_out/ops.log 2>&1; echo ops=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M.csv python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32 > gpurun_out/ncu.log 2>&1; echo ncu=$?
