python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -v warning | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -5
timeout 300 python tools/time_preint.py
