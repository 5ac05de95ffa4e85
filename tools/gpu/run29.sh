python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -iE " error" | head -3
timeout 300 python tools/fused_probe.py --config 3 --order 1 --width 4096 --height 4096 --reps 3
timeout 300 python tools/fused_probe.py --config 1 --order 1 --width 128 --height 128 --reps 20
timeout 300 python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 5
timeout 600 python tools/phase_profile.py --config 3 --order 1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
