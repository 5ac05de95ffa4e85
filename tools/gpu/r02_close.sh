# round-2 close on the restored tree (sources hash 5741203ee3e4): smoke, the
# default bench line, the reference arm, the order-4 tile kernel's DRAM traffic
# (metrics pass, then one ncu --set full capture of the same launch), the whole
# GPU suite last
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/c_bench_ref.json 2> gpurun_out/c_bench_ref.err; echo "ref rc=$?"
P="python tools/step_probe.py --order 4 --reps 0"
$P > gpurun_out/c_p4.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tile_kernel --csv --log-file gpurun_out/r02_r4_launches.csv $P > /dev/null 2>&1
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:tile_kernel -c 1 -o /tmp/r4 $P > /dev/null 2>&1; echo "ncu r4 rc=$?"
ncu -i /tmp/r4.ncu-rep --page raw --csv > gpurun_out/r02_r4_tile_raw.csv 2>/dev/null
ncu -i /tmp/r4.ncu-rep --page details --csv > gpurun_out/r02_r4_tile_details.csv 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c_tests.log
ls -la gpurun_out
