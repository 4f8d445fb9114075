mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -s -k "operators or batched" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python tools/profile_ops.py --gmres 0 --batches 1,32 > gpurun_out/ops.log 2>&1
python tools/profile_ops.py --gmres 0 --only "coarse solve" --reps 1 --batches 32 > gpurun_out/plain.log 2>&1 && ncu --set full --import-source on -k "regex:band_solve|xform_fft" -s 0 -c 2 -o gpurun_out/coarse_full python tools/profile_ops.py --gmres 0 --only "coarse solve" --reps 1 --batches 32 > gpurun_out/ncu.log 2>&1; echo ncu=$?
