timeout 900 python -m pytest tests/test_gpu_scan_tma.py tests/test_gpu_parity.py tests/test_gpu_strips.py tests/test_gpu_global.py -q -x 2>&1 | tail -3
timeout 300 python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 1 --reps 10 --anchor global 2>&1 | tail -5
