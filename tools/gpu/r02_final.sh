# round-2 evidence: smoke, GPU tests, the default bench line, ncu launch list
# of the r=1 step and one ncu --set full capture per timed kernel family,
# exported to CSV on the box (reports stay in /tmp: gpurun_out < 64 MiB)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 1500 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
P="python tools/step_probe.py --order 1 --reps 1"
$P > gpurun_out/p1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_r1_launches.csv $P > gpurun_out/p1n.log 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:"scan_|gx1_kernel" -s 9 -c 9 -o /tmp/r02_r1_full $P > gpurun_out/p2n.log 2>&1
ncu -i /tmp/r02_r1_full.ncu-rep --page raw --csv > gpurun_out/r02_r1_full_raw.csv 2>/dev/null
ncu -i /tmp/r02_r1_full.ncu-rep --page details --csv > gpurun_out/r02_r1_full_details.csv 2>/dev/null
P2="python tools/step_probe.py --order 2 --reps 1"
$P2 > gpurun_out/p3.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"fused_kernel" -s 1 -c 1 -o /tmp/r02_r2_fused $P2 > gpurun_out/p3n.log 2>&1
ncu -i /tmp/r02_r2_fused.ncu-rep --page raw --csv > gpurun_out/r02_r2_fused_raw.csv 2>/dev/null
ncu -i /tmp/r02_r2_fused.ncu-rep --page details --csv > gpurun_out/r02_r2_fused_details.csv 2>/dev/null
du -sh gpurun_out
