timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/t5_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/t5_bench.json 2>gpurun_out/t5_bench.err
cat gpurun_out/t5_pytest.log; cut -c1-1200 gpurun_out/t5_bench.json; tail -3 gpurun_out/t5_bench.err
