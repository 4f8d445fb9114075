mkdir -p gpurun_out
timeout 300 python tools/gmres_only.py 2049 300 64 20 > gpurun_out/gm20.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gm.csv python tools/gmres_only.py 2049 300 64 20 > gpurun_out/ncu_gm.log 2>&1; echo ncu=$?
