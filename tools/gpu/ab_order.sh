# A/B of the largest-first work order (BSF_ORDER=0: raster hand-out)
set -x
for i in 1 2; do
for o in 0 1; do
BSF_ORDER=$o python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 20
BSF_ORDER=$o python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 1 --reps 10
done; done
for o in 0 1; do
BSF_ORDER=$o python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 2 --reps 2
done
python tools/item_balance.py --config 2
python tools/item_balance.py --config 3 --order 1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
