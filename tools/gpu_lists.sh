# Launch lists (batch 32 / 1) with DRAM bytes, then ncu --set full of the kernels named in $KERNELS (regex list).
# Host setup + a kernel-name filter: the native setup's cuSOLVER eigen-solves launch ~15k small kernels.
mkdir -p gpurun_out
TAG=${TAG:-r02}
CMD="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 32 --setup host"
$CMD > gpurun_out/plain_$TAG.log 2>&1; echo plain=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M_$TAG.csv $CMD > /dev/null 2>&1; echo ncu32=$?
CMD1="python tools/profile_ops.py --gmres 0 --only M^-1 --reps 1 --batches 1 --setup host"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_M_b1_$TAG.csv $CMD1 > /dev/null 2>&1; echo ncu1=$?
for K in ${KERNELS:-local_dst_kernel band_solve_kernel xform_fft_kernel}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/full_${K}_$TAG $CMD > /dev/null 2>&1; echo full_$K=$?
done
