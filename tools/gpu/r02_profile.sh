# round-2 profiles of the bench workload (config 3): launch list of the r=1
# step, ncu --set full of the scans and gx1 (r=1) and of fused_kernel<2> (r=2)
set -x
P="python tools/step_probe.py --order 1 --reps 1"
$P > gpurun_out/p1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_r1_launches.csv $P > gpurun_out/p1n.log 2>&1
$P > gpurun_out/p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"scan_|gx1_kernel" -s 9 -c 9 -o gpurun_out/r02_r1_full $P > gpurun_out/p2n.log 2>&1
P2="python tools/step_probe.py --order 2 --reps 0"
$P2 > gpurun_out/p3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fused_kernel" -s 1 -c 1 -o gpurun_out/r02_r2_fused $P2 > gpurun_out/p3n.log 2>&1
tail -2 gpurun_out/p1n.log gpurun_out/p2n.log gpurun_out/p3n.log
