timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/t4_pytest.log
timeout 600 python bench.py > gpurun_out/t4_bench.json 2>gpurun_out/t4_bench.err
cat gpurun_out/t4_pytest.log; cat gpurun_out/t4_bench.json; tail -5 gpurun_out/t4_bench.err
