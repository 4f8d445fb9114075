# GPU tests + batch-1/32 timings + band configs at batch 32 + GMRES profile (n=2049).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log; grep "^cfg" gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_ops.py --gmres 0 --batches 1,32 2>&1 | grep "B="
for c in 0 7 8; do
  echo "cfg $c: $(HELM_BAND_CFG=$c timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve' --batches 32 2>&1 | grep -i 'coarse solve' | tail -1)"
done
timeout 600 python tools/gmres_profile.py 2049 300 64 50 > gpurun_out/gmres_prof.log 2>&1; echo gp=$?; tail -3 gpurun_out/gmres_prof.log
