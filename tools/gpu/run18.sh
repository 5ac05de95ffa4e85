for x in "" "-DBSF_EXP_NOSPLIT" "-DBSF_EXP_NOB" "-DBSF_EXP_NOSPLIT -DBSF_EXP_NOB"; do
  BSF_NVCC_EXTRA="$x" python -c "from paper_1109_5114_b200 import build as B; B.build(force=True)" 2>&1 | grep -iE " error" | head -3
  echo "variant [$x]"
  timeout 300 python tools/fused_probe.py --config 4 --order 3 --width 1024 --height 1024 --reps 1
done
