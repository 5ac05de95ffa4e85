for v in "" tools/libbsf_b.so tools/libbsf_e.so tools/libbsf_f.so; do
  echo "lib=$v"; BSF_LIB=$v timeout 300 python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 1 --reps 10 --anchor global
done
