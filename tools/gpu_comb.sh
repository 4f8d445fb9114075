timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python tools/profile_ops.py --gmres 0 --only 'local sum,M^-1' --batches 1,32 2>&1 | grep "B="
timeout 300 python tools/gmres_fixed.py 50 2>&1 | tail -1
timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
