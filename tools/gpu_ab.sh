# A/B: M^-1 timings with env toggles, alternating, same box
mkdir -p gpurun_out; : > gpurun_out/ab.log
for i in 1 2 3; do
  echo "A (default)" >> gpurun_out/ab.log; python tools/profile_ops.py --gmres 0 --reps 10 --only "M^-1" --batches 32 >> gpurun_out/ab.log 2>&1
  echo "B ($1)" >> gpurun_out/ab.log; env $1=1 python tools/profile_ops.py --gmres 0 --reps 10 --only "M^-1" --batches 32 >> gpurun_out/ab.log 2>&1
done
