# Round evidence: smoke, pytest -m gpu, bench (driver flags), reference arm, then the launch lists (batch 32 / 1)
# and ncu --set full captures of the top kernels (tools/gpu_lists.sh: host setup, so the profiled process
# launches only this library's kernels).
mkdir -p gpurun_out
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/smi_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu_$TAG.txt 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_gpu_$TAG.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
if [ "${REF:-1}" = "1" ]; then timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.log 2>&1; echo ref=$?; fi
KERNELS="${KERNELS:-local_dst_kernel band_tma_kernel xform_fft_kernel}" bash tools/gpu_lists.sh
