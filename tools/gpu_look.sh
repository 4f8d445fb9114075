# GMRES look-ahead on/off: GPU tests, bench GMRES lines (n=2049).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for e in 1 0; do
  echo "== LOOKAHEAD=$e"
  HELM_GMRES_LOOKAHEAD=$e timeout 900 python bench.py > gpurun_out/bench_look$e.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_look$e.log').read().strip().splitlines()[-1]); print(d['value'], d['gmres'])"
done
timeout 300 python tools/cfg4a_count.py 0 1 2>&1 | tail -1
