mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -s > gpurun_out/pytest_multi.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_multi.log
