# Determinism of the cfg4a count: repeated runs of one build/config.
for i in 1 2 3; do HELM_STRIP_COMP=0 timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1; done
for i in 1 2; do HELM_STRIP_COMP=3 timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "large_configs" 2>&1 | grep "^cfg\|passed\|failed"
