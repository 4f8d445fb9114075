# ncu --set full of one kernel (regex $1) during one SHS2 apply at config 5, batch 32
mkdir -p gpurun_out
python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32 > gpurun_out/plain.log 2>&1; echo plain=$?
ncu --set full --clock-control none --import-source on -k "regex:$1" -s 1 -c 1 -o gpurun_out/k_$1 python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32 > gpurun_out/ncu_$1.log 2>&1; echo ncu=$?
