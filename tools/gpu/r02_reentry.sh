# re-entry validation of the restored tree: smoke, whole GPU suite, default bench
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/re_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/re_tests.log
timeout 1500 python bench.py > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err; echo "bench rc=$?"
