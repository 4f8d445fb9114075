# State check after a re-entry: smoke, bench (default flags), the GMRES setup probe, then the GPU tests.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
S=$(date +%s); timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$? $(( $(date +%s) - S ))s
tail -c 6000 gpurun_out/bench.log
timeout 600 python tools/gmres_setup_ab.py > gpurun_out/gmres_setup.log 2>&1; echo gm=$?
cat gpurun_out/gmres_setup.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
