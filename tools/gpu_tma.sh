# TMA-staged band kernel: A/B against the cp.async kernel (outputs must be bitwise equal), coarse-solve tests.
mkdir -p gpurun_out
AB=tma timeout 900 python tools/strip_first_ab.py > gpurun_out/tma_ab.log 2>&1; echo ab=$?
cat gpurun_out/tma_ab.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -m gpu -x -q -k "segmented or compact or operators_match or batched or multi" > gpurun_out/tma_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/tma_pytest.log
