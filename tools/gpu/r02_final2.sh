# final round-2 evidence on the committed sources: smoke, GPU tests, the
# default bench line, a config-4 frame, the order-1 launch list, ncu --set full
# captures of the scans + gx1 (order 1) and fused_kernel<2>/<3> (orders 2/3)
# with their SASS source pages (reports stay in /tmp)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/f_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/f_tests.log
timeout 1500 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --config 4 --frames-per-gpu 1 --steps 1 > gpurun_out/f_c4.json 2> gpurun_out/f_c4.err; echo "c4 rc=$?"
P="python tools/step_probe.py --order 1 --reps 1"
$P > gpurun_out/f_p1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_r1_launches.csv $P > /dev/null 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:"scan_|gx1_kernel" -s 9 -c 9 -o /tmp/r1 $P > /dev/null 2>&1
ncu -i /tmp/r1.ncu-rep --page raw --csv > gpurun_out/r02_r1_full_raw.csv 2>/dev/null
ncu -i /tmp/r1.ncu-rep --page details --csv > gpurun_out/r02_r1_full_details.csv 2>/dev/null
ncu -i /tmp/r1.ncu-rep --page source --csv --print-source sass --kernel-name regex:gx1_kernel > gpurun_out/r02_gx1_source_sass.csv 2>/dev/null
for R in 2 3; do
P="python tools/step_probe.py --order $R --reps 1"
$P > gpurun_out/f_p$R.log 2>&1 || continue
ncu -f --set full --clock-control none --import-source on -k regex:fused_kernel -s 1 -c 1 -o /tmp/f$R $P > /dev/null 2>&1
ncu -i /tmp/f$R.ncu-rep --page raw --csv > gpurun_out/r02_r${R}_fused_raw.csv 2>/dev/null
ncu -i /tmp/f$R.ncu-rep --page details --csv > gpurun_out/r02_r${R}_fused_details.csv 2>/dev/null
ncu -i /tmp/f$R.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_f${R}_source_sass.csv 2>/dev/null
done
du -sh gpurun_out; ls -la gpurun_out
