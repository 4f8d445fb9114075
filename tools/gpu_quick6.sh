# Quick check after a local-kernel change: per-op timings, DST-vs-dense test, operator parity tests.
mkdir -p gpurun_out
timeout 600 python tools/profile_ops.py --gmres 0 --reps 5 --batches 1,32 > gpurun_out/q6_ops.log 2>&1; cat gpurun_out/q6_ops.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large_parity.py -m gpu -x -q -k "fast_sine or operators_match or weights_before or maximal" > gpurun_out/q6_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/q6_pytest.log
