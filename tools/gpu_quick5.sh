# Quick A/B: coarse-solve / M^-1 timings with HELM_FFT_MINB=1 and 2 (band forward unroll in both), per-op timings.
mkdir -p gpurun_out
for mb in 1 2; do
  HELM_FFT_MINB=$mb HELM_STRIP_FIRST=1 timeout 600 python tools/strip_first_ab.py new > gpurun_out/q5_minb$mb.log 2>&1; echo minb$mb=$?
  cat gpurun_out/q5_minb$mb.log
done
timeout 600 python tools/profile_ops.py --gmres 0 --reps 5 --batches 1,32 > gpurun_out/q5_ops.log 2>&1; cat gpurun_out/q5_ops.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "segmented or compact or operators_match or batched" > gpurun_out/q5_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/q5_pytest.log
