# PDL (implicit trigger) on/off with look-ahead: fixed GMRES, batch-1/32 M^-1; seg prefetch variants.
for e in "HELM_PDL=1" "HELM_PDL=0"; do
  echo "== $e"; env $e timeout 300 python tools/gmres_fixed.py 50 2>&1 | tail -1
  env $e timeout 300 python tools/profile_ops.py --gmres 0 --only 'M^-1,coarse solve' --batches 1,32 2>&1 | grep "B="
done
for pf in 0 1 2; do echo "seg pf $pf: $(HELM_SEG_PF=$pf timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve' --batches 1 2>&1 | grep 'B=')"; done
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
