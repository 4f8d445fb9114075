# cfg4a iteration count vs coarse-solve path / accuracy.
for a in "0 1" "1 1" "0 2" "2 1"; do timeout 300 python tools/cfg4a_count.py $a 2>&1 | tail -1; done
HELM_BAND_SEG_MAX=0 timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
HELM_BAND_SEG_MAX=0 timeout 300 python tools/cfg4a_count.py 1 1 2>&1 | tail -1
