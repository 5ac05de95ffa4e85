# banded scans in bsf_run_host: bit-identity checks, then the order-1 bench line (e2e)
set -x
python tools/diag_banded.py > gpurun_out/diag.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_global.py -q -x > gpurun_out/banded_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py --orders 1 --no-cpu-baseline > gpurun_out/banded_bench.json 2> gpurun_out/banded_bench.err; echo "bench rc=$?"
