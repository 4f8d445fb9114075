# Round-2 evidence: smoke, pytest -m gpu, bench (driver flags), reference arm, launch lists (batch 32 / 1),
# ncu --set full of the top kernel, SASS instruction mix of the library.
mkdir -p gpurun_out
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/smi_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu_$TAG.txt 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_gpu_$TAG.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
if [ "${REF:-1}" = "1" ]; then timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.log 2>&1; echo ref=$?; fi
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32"
$CMD > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M_$TAG.csv $CMD > /dev/null 2>&1; echo ncu32=$?
CMD1="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 1"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M_b1_$TAG.csv $CMD1 > /dev/null 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:local_fdm_dmma -s 1 -c 1 -o gpurun_out/top_kernel_$TAG $CMD > /dev/null 2>&1; echo ncufull=$?
