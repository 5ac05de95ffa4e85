# last validation on the final sources: the whole GPU suite (incl. the i8
# tcgen05 prototype's exactness test) and the extended fuzz
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/l_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/l_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/l_tests.log
timeout 2400 python tools/fuzz_extended.py > gpurun_out/l_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -2 gpurun_out/l_fuzz.log
