for x in "" "-DBSF_R3_TWO_LIMB"; do
  BSF_NVCC_EXTRA="$x" python -c "from paper_1109_5114_b200 import build as B; B.build(force=True)" 2>&1 | grep -iE " error" | head -3
  echo "variant [$x]"
  timeout 300 python tools/fused_probe.py --config 4 --order 3 --width 1024 --height 1024 --reps 1
  timeout 300 python tools/fused_probe.py --config 3 --order 3 --width 1024 --height 1024 --reps 1
  timeout 300 python tools/fused_probe.py --config 5 --order 3 --width 1024 --height 1024 --reps 1
done
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_orders.py -q -x 2>&1 | tail -3
