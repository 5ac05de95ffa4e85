set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/v_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/v_tests.log
timeout 1500 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo "bench rc=$?"
