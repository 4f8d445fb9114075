# L2 bulk prefetch of the band factors during the forward FFT: on/off.
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for e in 1 0; do
  echo "== HELM_L2_PREFETCH=$e"
  HELM_L2_PREFETCH=$e timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve,M^-1' --batches 1,8,32 2>&1 | grep "B="
  HELM_L2_PREFETCH=$e timeout 300 python tools/gmres_fixed.py 50 2>&1 | tail -1
done
