# Quick A/B loop: operator parity tests + a short bench (no CPU leg, no GMRES).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large_parity.py -q -x -k "operators or maximal or weights" > gpurun_out/quick_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/quick_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --gmres 0 --no-cpu > gpurun_out/quick_bench.log 2>&1; echo bench=$?
python - <<'PY'
import json
l=[x for x in open('gpurun_out/quick_bench.log') if x.startswith('{')]
d=json.loads(l[-1]); print('value', d['value'], 'ms', d['ms_per_step']); print({k:v['ms_per_batch'] for k,v in d['phases'].items()})
PY
