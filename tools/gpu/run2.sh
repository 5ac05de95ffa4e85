# fused split-contraction path: tile tests + bench A/B
timeout 900 python -m pytest tests/test_gpu_tile.py -x -q 2>&1 | tail -15 > gpurun_out/t2_pytest.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --precision dd --anchor tile > gpurun_out/t2_bench_fused.json 2>gpurun_out/t2_bench_fused.err
cat gpurun_out/t2_pytest.log; tail -c 1500 gpurun_out/t2_bench_fused.json; tail -5 gpurun_out/t2_bench_fused.err
