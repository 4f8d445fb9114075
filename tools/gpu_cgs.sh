mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python tools/gmres_profile.py 2049 300 64 50 > gpurun_out/gmres_prof.log 2>&1; echo gp=$?
timeout 300 python tools/gmres_trace.py 50 2 > gpurun_out/gtrace.log 2>&1; echo tr=$?
