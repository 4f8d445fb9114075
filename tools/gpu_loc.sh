mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python tools/profile_ops.py --batches 1,32 --gmres 0 > gpurun_out/ops.log 2>&1; echo ops=$?
