python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -iE " error" | head -3
for st in 32 64; do
  echo "stile $st"
  BSF_STILE=$st timeout 300 python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 5
  BSF_STILE=$st timeout 300 python tools/fused_probe.py --config 3 --order 1 --width 4096 --height 4096 --reps 3
  BSF_STILE=$st timeout 300 python tools/fused_probe.py --config 3 --order 2 --width 2048 --height 2048 --reps 2
  BSF_STILE=$st timeout 300 python tools/fused_probe.py --config 1 --order 1 --width 128 --height 128 --reps 20
  BSF_STILE=$st timeout 300 python tools/fused_probe.py --config 4 --order 3 --width 1024 --height 1024 --reps 1
done
BSF_STILE=64 timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_orders.py tests/test_gpu_tile.py -q -x 2>&1 | tail -3
