# super-tile rule check: config 3 r = 2 (u8, plain run 64 x 64; split passes 32 x 32)
python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 2 --reps 1 --split 2
python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 2 --reps 1 --split 2 --super-tile 32
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_alg1.py -q -x 2>&1 | tail -3
