# Multi-RHS GMRES tests + bench GMRES numbers under PDL / look-ahead toggles.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/pytest_multi.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_multi.log
for e in "X=1" "HELM_GMRES_LOOKAHEAD=0" "HELM_PDL=0"; do
  env $e timeout 900 python bench.py --no-cpu > gpurun_out/bench_t.log 2>&1
  echo "$e: $(python -c "import json; d=json.loads(open('gpurun_out/bench_t.log').read().strip().splitlines()[-1]); g=d['gmres']; print(d['value'], g['seconds'], g['fixed_ms_per_iter'])")"
done
