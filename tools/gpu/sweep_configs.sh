# N=1 throughput of the fused product path on every BASELINE config (bench.py
# lines; config 4 = one 2048^2 frame channel per step, config 5 not run at
# full size here: see tools/fused_probe.py crops)
python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -iE " error" | head -3
for co in "1 1" "2 2" "3 1" "3 2" "3 3" "4 3"; do
  set -- $co
  steps=5; [ "$2" = "3" ] && steps=1
  timeout 600 python bench.py --config $1 --order $2 --steps $steps --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1
done > gpurun_out/sweep_configs.jsonl
for c in 5; do
  timeout 600 python tools/fused_probe.py --config $c --order 3 --width 4096 --height 2048 --reps 1
done > gpurun_out/sweep_c5.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
