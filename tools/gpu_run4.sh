mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -k "operators or batched or zero or dimension or csr" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python tools/profile_ops.py --gmres 0 --batches 32 > gpurun_out/ops.log 2>&1; echo ops=$?
CMD="python tools/profile_ops.py --gmres 0 --only 'local sum' --reps 1 --batches 32"
eval $CMD > gpurun_out/plain.log 2>&1 && eval ncu --set full --import-source on -k regex:local_fdm_fast -s 2 -c 1 -o gpurun_out/local_fast $CMD > gpurun_out/ncu.log 2>&1; echo rc=$?
