mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32"
eval $CMD > gpurun_out/plain.log 2>&1 && eval ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu=$?
