# GMRES-focused check: all GPU tests, then the bench's GMRES section.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gm.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gm.log
grep -E "^cfg3|^cfg4a|^cfg2|cfg4b" gpurun_out/pytest_gm.log | head
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/gm_bench.log 2>&1; echo bench=$?
python - <<'PY'
import json
l=[x for x in open('gpurun_out/gm_bench.log') if x.startswith('{')]
d=json.loads(l[-1]); print('value', d['value']); g=d['gmres']; print({k:g[k] for k in ('iterations','iter_per_s','fixed_iter_per_s','fixed_ms_per_iter')}); print(g['roofline']); print(g['multi'])
PY
