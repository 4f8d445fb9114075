# ncu of the three CGS sweeps (K1 cgs_dots, K2 cgs_update_dots, K3 cgs_final) in a fixed 50-iteration
# GMRES run at config 5: launch list with DRAM bytes, plus --set full of each kernel at iteration ~49.
mkdir -p gpurun_out
CMD="python tools/gmres_fixed.py 50"
$CMD > gpurun_out/gmfix.log 2>&1; echo plain=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:cgs_ --csv --log-file gpurun_out/launches_cgs.csv python tools/gmres_fixed.py 50 > /dev/null 2>&1; echo list=$?
for K in cgs_dots cgs_update_dots cgs_final; do
  ncu --set full --clock-control none -k regex:$K -s 48 -c 1 -o gpurun_out/k_$K python tools/gmres_fixed.py 50 > /dev/null 2>&1; echo $K=$?
done
