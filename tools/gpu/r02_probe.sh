BSF_LIB=tools/libbsf_gray.so timeout 900 python -m pytest tests/test_gpu_global.py -q -x 2>&1 | tail -2
for v in "" tools/libbsf_gray.so; do
  echo "lib=$v"; BSF_LIB=$v timeout 300 python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 1 --reps 10 --anchor global
done
