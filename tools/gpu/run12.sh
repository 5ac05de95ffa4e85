python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -v warning | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -5
timeout 300 python tools/time_preint.py
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,lts__t_bytes.sum --clock-control none --csv python tools/scan_probe.py 1 > gpurun_out/scan_ncu.csv 2> gpurun_out/scan_ncu.err
tail -3 gpurun_out/scan_ncu.err
