BSF_STILE=64 timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_orders.py tests/test_gpu_tile.py -q -x 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
