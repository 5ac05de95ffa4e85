timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/t6_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/t6_bench.json 2>gpurun_out/t6_bench.err
python tools/phase_profile.py > gpurun_out/t6_phase.log 2>&1
cat gpurun_out/t6_pytest.log gpurun_out/t6_phase.log; cut -c1-400 gpurun_out/t6_bench.json; tail -3 gpurun_out/t6_bench.err
