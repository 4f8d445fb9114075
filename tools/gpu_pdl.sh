# PDL on/off: GPU tests, batch-1/32 timings, GMRES profile (n=2049).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for e in 1 0; do
  echo "== HELM_PDL=$e"
  HELM_PDL=$e timeout 300 python tools/profile_ops.py --gmres 0 --batches 1,32 2>&1 | grep "B="
  HELM_PDL=$e timeout 600 python tools/gmres_profile.py 2049 300 64 50 2>&1 | tail -1
done
timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
