# round-2 closing evidence on the final sources: the fuzz tests (new error
# reading R26), the default bench line, the order-1 launch list, ncu --set full
# captures of the scans + gx1 (order 1) and fused_kernel<2>/<3> (orders 2/3)
# for the traffic figures bench.py reports (profiles/r02_traffic.json)
set -x
timeout 1200 python -m pytest tests/test_gpu_fuzz.py -m gpu -q > gpurun_out/z_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -2 gpurun_out/z_fuzz.log
P="python tools/step_probe.py --order 1 --reps 1"
$P > gpurun_out/z_p1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_r1_launches.csv $P > /dev/null 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:"scan_|gx1_kernel" -s 9 -c 9 -o /tmp/r1 $P > /dev/null 2>&1
ncu -i /tmp/r1.ncu-rep --page raw --csv > gpurun_out/r02_r1_full_raw.csv 2>/dev/null
ncu -i /tmp/r1.ncu-rep --page details --csv > gpurun_out/r02_r1_full_details.csv 2>/dev/null
for R in 2 3; do
P="python tools/step_probe.py --order $R --reps 1"
$P > gpurun_out/z_p$R.log 2>&1 || continue
ncu -f --set full --clock-control none --import-source on -k regex:fused_kernel -s 1 -c 1 -o /tmp/f$R $P > /dev/null 2>&1
ncu -i /tmp/f$R.ncu-rep --page raw --csv > gpurun_out/r02_r${R}_fused_raw.csv 2>/dev/null
ncu -i /tmp/f$R.ncu-rep --page details --csv > gpurun_out/r02_r${R}_fused_details.csv 2>/dev/null
done
timeout 1500 python bench.py > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err; echo "bench rc=$?"
du -sh gpurun_out; ls -la gpurun_out
