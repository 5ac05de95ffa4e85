set -x
timeout 1800 python -m pytest tests/test_gpu_strips.py tests/test_gpu_global.py tests/test_gpu_fused.py tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x 2>&1 | tail -12
