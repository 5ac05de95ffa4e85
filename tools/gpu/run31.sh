for np in 2 3 5; do
  BSF_NVCC_EXTRA="-DBSF_G3_NP2=$np" python -c "from paper_1109_5114_b200 import build as B; B.build(force=True, verbose=True)" 2>&1 | grep -A2 "fused_kernelILi3" | grep -E "spill|Used"
  echo "NP2=$np"
  timeout 300 python tools/fused_probe.py --config 4 --order 3 --width 1024 --height 1024 --reps 1
  timeout 300 python tools/fused_probe.py --config 5 --order 3 --width 1024 --height 1024 --reps 1
done
python -c "from paper_1109_5114_b200 import build as B; B.build(force=True)" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_orders.py -q -x 2>&1 | tail -2
