python -c "from paper_1109_5114_b200 import build as B; B.build()" >/dev/null 2>&1
for o in 1 2 3; do timeout 300 python tools/fused_probe.py --config 2 --order $o --width 1024 --height 1024 --reps 2; done
for n in 2 3 4; do timeout 300 python tools/fused_probe.py --config 2 --order 1 --split $n --width 1024 --height 1024 --reps 3; done
timeout 300 python tools/fused_probe.py --config 2 --order 2 --split 2 --width 1024 --height 1024 --reps 3
