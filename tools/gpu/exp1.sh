for e in 0 1 2; do
  BSF_NVCC_EXTRA="-DBSF_EXPERIMENT=$e" python -c "from paper_1109_5114_b200 import build as B; B.build(force=True)"
  echo "== experiment $e"; python tools/phase_profile.py 2>&1 | grep -E "gather|pre-int|keys"
done
