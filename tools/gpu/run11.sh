python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -v warning | tail -2
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,lts__t_bytes.sum --clock-control none --csv python tools/scan_probe.py 1 > gpurun_out/scan_ncu.csv 2> gpurun_out/scan_ncu.err
tail -3 gpurun_out/scan_ncu.err
