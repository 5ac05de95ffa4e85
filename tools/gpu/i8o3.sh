set -x
timeout 900 python -m pytest tests/test_gpu_i8_order3.py -q -x > gpurun_out/i8o3_tests.log 2>&1; echo "tests rc=$?"
