python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -iE " error" | head -3
timeout 300 python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 5
timeout 300 python tools/fused_probe.py --config 3 --order 2 --width 4096 --height 4096 --reps 1
timeout 300 python tools/fused_probe.py --config 3 --order 1 --width 4096 --height 4096 --reps 3
timeout 300 python tools/fused_probe.py --config 5 --order 3 --width 1024 --height 1024 --reps 1
timeout 600 python tools/phase_profile.py --config 3 --order 2
timeout 1500 python -m pytest tests/test_gpu_fused.py tests/test_gpu_strips.py tests/test_gpu_tile.py tests/test_gpu_orders.py -q -x 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
