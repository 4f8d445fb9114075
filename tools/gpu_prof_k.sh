# usage: bash tools/gpu_prof_k.sh <kernel-regex> <profile_ops --only> <batches> <skip>
mkdir -p gpurun_out
python tools/profile_ops.py --gmres 0 --only "$2" --reps 1 --batches $3 > gpurun_out/plain.log 2>&1 && ncu --set full --import-source on -k "regex:$1" -s $4 -c 1 -o gpurun_out/kprof python tools/profile_ops.py --gmres 0 --only "$2" --reps 1 --batches $3 > gpurun_out/ncu.log 2>&1; echo ncu=$?
