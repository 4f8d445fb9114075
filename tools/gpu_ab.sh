# A/B of an environment switch: quick tests, then bench (no CPU leg, no GMRES) with and without it.
# usage: VAR=HELM_FFT16 bash tools/gpu_ab.sh
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large_parity.py -q -x -k "operators or maximal or weights" > gpurun_out/quick_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/quick_tests.log
for v in 1 0 1 0; do
  env $VAR=$v python bench.py --steps 10 --warmup 3 --gmres 0 --no-cpu 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', d['value'], d['ms_per_step'], {k: v['ms_per_batch'] for k, v in d['phases'].items()})"
done
env $VAR=1 python tools/profile_ops.py --gmres 0 --only M^-1 --reps 20 --batches 1 2>/dev/null | tail -3
env $VAR=0 python tools/profile_ops.py --gmres 0 --only M^-1 --reps 20 --batches 1 2>/dev/null | tail -3
