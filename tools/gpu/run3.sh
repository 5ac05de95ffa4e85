timeout 900 python -m pytest tests/test_gpu_tile.py -x -q 2>&1 | tail -15 > gpurun_out/t3_pytest.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --anchor tile > gpurun_out/t3_bench.json 2>gpurun_out/t3_bench.err
python tools/phase_profile.py > gpurun_out/t3_phase.log 2>&1
cat gpurun_out/t3_pytest.log gpurun_out/t3_phase.log; tail -c 1500 gpurun_out/t3_bench.json; tail -5 gpurun_out/t3_bench.err
