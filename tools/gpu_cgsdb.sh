# CGS2 double-buffered stage on/off: GPU tests, CGS2 per-j timings, fixed GMRES.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
for e in 1 0; do
  echo "== HELM_CGS_DB=$e"
  HELM_CGS_DB=$e timeout 600 python tools/gmres_profile.py 2049 300 64 50 2>&1 | grep "CGS2"
  HELM_CGS_DB=$e timeout 300 python tools/gmres_fixed.py 50 2>&1 | tail -1
done
