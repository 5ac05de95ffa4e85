# A/B of the largest-first work order (work_order = 0: raster hand-out)
set -x
for i in 1 2; do
for o in 0 1; do
python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 20 --opt work_order=$o
python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 1 --reps 10 --opt work_order=$o
done; done
for o in 0 1; do
python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 2 --reps 2 --opt work_order=$o
done
python tools/item_balance.py --config 2
python tools/item_balance.py --config 3 --order 1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
