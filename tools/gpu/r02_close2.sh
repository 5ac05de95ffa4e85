# after r02_close.sh: the default bench line with the order-4 traffic figure in
# place (profiles/r02_traffic.json re-keyed), then new fuzz seeds while the box
# is there
set -x
timeout 1200 python bench.py > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err; echo "bench rc=$?"
timeout 780 python tools/fuzz_extended.py --shift 2000 > gpurun_out/d_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -3 gpurun_out/d_fuzz.log
