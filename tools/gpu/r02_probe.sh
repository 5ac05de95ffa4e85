for v in "" _v1 "" _v1; do
  echo "== libbsf$v"
  BSF_LIB=paper_1109_5114_b200/libbsf$v.so timeout 300 python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 1 --reps 20 --anchor global 2>&1 | tail -1
done
cp paper_1109_5114_b200/libbsf_v1.so paper_1109_5114_b200/libbsf.so
timeout 900 python -m pytest tests/test_gpu_global.py tests/test_gpu_fuzz.py -q -x -k "global" 2>&1 | tail -2
