# config 2 timing (3 repeats) + fused/parity tests
for i in 1 2 3; do python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 20; done
python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 2 --reps 2
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
