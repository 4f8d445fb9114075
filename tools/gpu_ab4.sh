# GPU tests (with cfg counts) + batch-1/32 timings + cfg4a count under the lane band path + launch list b1.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log; grep "^cfg" gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_ops.py --gmres 0 --batches 1,32 2>&1 | grep "B="
HELM_BAND_SEG_MAX=0 timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 1"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M_b1.csv $CMD > gpurun_out/ncu_b1.log 2>&1; echo ncu=$?
