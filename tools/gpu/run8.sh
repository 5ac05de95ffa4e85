timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/t8_pytest.log
bash tools/gpu/profile_round.sh > /dev/null 2>&1
cat gpurun_out/t8_pytest.log; cut -c1-300 gpurun_out/prof_bench.json; cat gpurun_out/prof_phase.log
