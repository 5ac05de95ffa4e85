# round-2 check: GPU tests, then the default bench line (config 3, orders 1-4)
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 1500 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_bench.json
