timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve,M^-1' --batches 1 2>&1 | grep "B="
timeout 300 python tools/gmres_fixed.py 50 2>&1 | tail -1
timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
HELM_BAND_SEG_MAX=0 timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
