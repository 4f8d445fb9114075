mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python tools/profile_ops.py --gmres 30 > gpurun_out/ops.log 2>&1; echo ops=$?
