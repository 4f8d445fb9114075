# Quick confirmation run: gpu tests + bench (ours) on one B200.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/smi.txt
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
