set -x
timeout 900 python -m pytest tests/test_gpu_global.py -q -x 2>&1 | tail -5
timeout 300 python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 1 --reps 10 --anchor global
BSF_LIB=tools/libbsf_minb1.so timeout 300 python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 1 --reps 10 --anchor global
timeout 300 python tools/time_preint.py 2>&1 | tail -5
