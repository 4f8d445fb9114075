# A/B of the fast-sine / edge box kernels against the DMMA / dense ones, the GMRES setup probe, then the GPU tests.
mkdir -p gpurun_out
timeout 600 python tools/gmres_setup_ab.py > gpurun_out/gmres_setup.log 2>&1; echo gm=$?
cat gpurun_out/gmres_setup.log
timeout 900 python tools/dst_ab.py > gpurun_out/dst_ab.log 2>&1; echo dst_ab=$?
cat gpurun_out/dst_ab.log | tail -8
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast_sine or operators_match or gmres_matches" > gpurun_out/pytest_parity.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_parity.log
