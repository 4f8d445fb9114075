# Strip-first coarse solve: A/B against the round-1 pass order, the GPU tests that touch the coarse solve, bench,
# then the launch lists / ncu captures (tools/gpu_lists.sh).
mkdir -p gpurun_out
timeout 900 python tools/strip_first_ab.py > gpurun_out/sf_ab.log 2>&1; echo ab=$?
cat gpurun_out/sf_ab.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_large_parity.py -m gpu -x -q > gpurun_out/pytest_sf.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_sf.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_sf.log 2>&1; echo bench=$?
grep -o '"value": [0-9.]*\|"phases": {[^}]*}[^}]*}[^}]*}[^}]*}[^}]*}[^}]*}\|"parity": {[^}]*}' gpurun_out/bench_sf.log
bash tools/gpu_lists.sh
