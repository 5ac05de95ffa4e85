python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -iE "error" | head -3
timeout 900 python -m pytest tests/test_gpu_strips.py tests/test_gpu_parity.py -q -x 2>&1 | tail -15
