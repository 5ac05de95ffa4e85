CMD="python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 1 --reps 1 --anchor global"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gx1_kernel -s 1 -c 1 -o gpurun_out/r02_gx1 $CMD > gpurun_out/ncu_gx1.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_gx1_launches.csv $CMD > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu_gx1.log
