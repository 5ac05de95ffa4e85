timeout 1500 python -m pytest tests/test_gpu_tile.py tests/test_gpu_fused.py tests/test_gpu_orders.py -q -x 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | cut -c1-300
python tools/phase_profile.py 2>&1 | grep -E "gather|pre-int|keys"
python tools/phase_profile.py --config 3 --order 2 2>&1 | grep -E "gather|pre-int|keys"
