# A/B: compact no-pivot band factors, L2 persisting window, split strip kernels (n=2049).
mkdir -p gpurun_out
python -c "import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)" 
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
for env in "X=1" "HELM_L2_PERSIST=0" "HELM_BAND_NOPIV=0 HELM_L2_PERSIST=0"; do
  echo "== $env"
  env $env timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve,M^-1' --batches 1,32 2>&1 | grep "B="
done
timeout 600 python tools/gmres_profile.py 2049 300 64 50 > gpurun_out/gmres_prof.log 2>&1; echo gp=$?; tail -3 gpurun_out/gmres_prof.log
