for s in 4 8; do echo "smb $s: $(HELM_SEG_SMB=$s timeout 300 python tools/profile_ops.py --gmres 0 --only 'coarse solve,M^-1' --batches 1 2>&1 | grep 'B=' | tr '\n' ' ')"; done
timeout 300 python tools/gmres_fixed.py 50 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "band or large" 2>&1 | tail -1
