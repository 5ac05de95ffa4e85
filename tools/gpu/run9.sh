set -x
for m in 2 1; do
  BSF_NVCC_EXTRA="-DBSF_MT3=$m" python -c "from paper_1109_5114_b200 import build as B; B.build(force=True)" 2>&1 | grep -v warning | tail -2
  echo "MT3=$m"
  timeout 400 python tools/phase_profile.py --config 4 --order 3 2>&1 | tail -25
done
python -c "from paper_1109_5114_b200 import build as B; B.build(force=True)" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_orders.py tests/test_gpu_strips.py -q -x 2>&1 | tail -5
