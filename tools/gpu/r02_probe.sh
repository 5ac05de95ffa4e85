P="python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 1 --reps 20 --anchor global"
for i in 1 2; do
  echo "wide:"; $P 2>&1 | tail -1
  echo "limb3:"; BSF_LIB=paper_1109_5114_b200/libbsf_w0.so $P 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gpu_global.py -q -x 2>&1 | tail -2
