# Fused strip partials in the band passes (batch >= 5): tests, timings, launch list b32.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve,M^-1' --batches 1,8,32 2>&1 | grep "B="
timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
HELM_BAND_SEG_MAX=0 timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
