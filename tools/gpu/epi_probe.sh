# Timing of the r = 2 MMA loop without the polynomial epilogue (diagnostics
# build, wrong results; fallback disabled so both runs do the same work)
python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 20 --opt split_tol=1e300
BSF_NVCC_EXTRA=-DBSF_DBG_NO_EPI python -m paper_1109_5114_b200.build -f > /dev/null 2>&1
python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 20 --opt split_tol=1e300
python -m paper_1109_5114_b200.build -f > /dev/null 2>&1
