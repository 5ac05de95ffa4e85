# sweep strip-scan shapes: NW RPW ND for int64 and dd
for cfg in "8 4 8 4 8 4" "8 8 4 4 16 2" "8 16 2 4 16 3" "4 16 4 8 8 3" "16 4 4 8 4 4"; do
  set -- $cfg
  BSF_NVCC_EXTRA="-DBSF_SCAN_NW_I64=$1 -DBSF_SCAN_RPW_I64=$2 -DBSF_SCAN_ND_I64=$3 -DBSF_SCAN_NW_DD=$4 -DBSF_SCAN_RPW_DD=$5 -DBSF_SCAN_ND_DD=$6" python -c "from paper_1109_5114_b200 import build as B; B.build(force=True)" 2>&1 | grep -iE "error" | head -3
  echo "cfg $cfg"
  timeout 300 python tools/time_preint.py 2>&1 | head -3
done
