for x in "" "-DBSF_EXP_NOB2" "-DBSF_EXP_NOA2" "-DBSF_EXP_NOA2 -DBSF_EXP_NOB2"; do
  BSF_NVCC_EXTRA="$x" python -c "from paper_1109_5114_b200 import build as B; B.build(force=True)" 2>&1 | grep -iE " error" | head -3
  echo "variant [$x]"
  timeout 300 python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 5
  timeout 300 python tools/fused_probe.py --config 3 --order 2 --width 2048 --height 2048 --reps 2
done
