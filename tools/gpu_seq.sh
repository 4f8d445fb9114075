# Sequential segment chains in band_seg (HELM_SEG_SCAN=1 default) vs Kogge-Stone (0).
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for e in 1 0; do
  echo "== HELM_SEG_SCAN=$e"
  HELM_SEG_SCAN=$e timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve,M^-1' --batches 1 2>&1 | grep "B="
  HELM_SEG_SCAN=$e timeout 300 python tools/gmres_fixed.py 50 2>&1 | tail -1
  HELM_SEG_SCAN=$e timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
done
