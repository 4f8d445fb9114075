for e in "HELM_PDL=1 HELM_GMRES_LOOKAHEAD=1" "HELM_PDL=0 HELM_GMRES_LOOKAHEAD=1" "HELM_PDL=1 HELM_GMRES_LOOKAHEAD=0" "HELM_PDL=0 HELM_GMRES_LOOKAHEAD=0"; do
  echo "== $e"; env $e timeout 300 python tools/gmres_fixed.py 50 2>&1 | tail -2
done
echo "== trace PDL=1"; HELM_PDL=1 HELM_GMRES_TRACE=1 timeout 300 python tools/gmres_fixed.py 50 2>&1 | grep "gmres it" | tail -60 | awk 'NR%10==0'
echo "== trace PDL=0"; HELM_PDL=0 HELM_GMRES_TRACE=1 timeout 300 python tools/gmres_fixed.py 50 2>&1 | grep "gmres it" | tail -60 | awk 'NR%10==0'
