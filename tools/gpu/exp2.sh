for m in 2 4; do
  BSF_NVCC_EXTRA="-DBSF_MT1=$m" python -c "from paper_1109_5114_b200 import build as B; B.build(force=True)"
  echo "MT1=$m"; python bench.py --config 3 --order 1 --steps 3 --no-cpu-baseline 2>/dev/null | cut -c1-150
  python bench.py --config 1 --steps 10 --no-cpu-baseline 2>/dev/null | cut -c1-150
done
