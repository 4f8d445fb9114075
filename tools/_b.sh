timeout 300 python tools/profile_ops.py --gmres 0 --reps 5 --batches 8,32 --only "coarse solve,M^-1" --setup host 2>&1 | grep "B="
timeout 600 python -m pytest tests/test_gpu_coarse_paths.py -m gpu -x -q > gpurun_out/b_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/b_pytest.log
