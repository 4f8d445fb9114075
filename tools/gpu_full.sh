# Round-end style evidence run: tests, smoke, bench (ours + reference arm), ncu launch lists (batch 32 and 1), ncu full of the top kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu=$?
CMD1="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 1"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M_b1.csv $CMD1 > gpurun_out/ncu_b1.log 2>&1; echo ncu_b1=$?
ncu --set full --clock-control none --import-source on -k regex:local_fdm_dmma -s 1 -c 1 -o gpurun_out/top_kernel $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
