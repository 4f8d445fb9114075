# Batch-1 costs at n=2049: per-operator timings, GMRES per-iteration pieces, ncu launch list of one M^-1 at batch 1.
mkdir -p gpurun_out
timeout 600 python tools/profile_ops.py --batches 1 --gmres 0 > gpurun_out/ops_b1.log 2>&1; echo ops=$?
timeout 600 python tools/gmres_profile.py 2049 300 64 50 > gpurun_out/gmres_prof.log 2>&1; echo gp=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M_b1.csv python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 1 > gpurun_out/ncu_b1.log 2>&1; echo ncu=$?
timeout 300 python tools/gmres_only.py 2049 300 64 20 > gpurun_out/gm20.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gm.csv python tools/gmres_only.py 2049 300 64 20 > gpurun_out/ncu_gm.log 2>&1; echo ncu=$?
