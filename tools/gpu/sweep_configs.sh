# N=1 throughput of the fused product path on the BASELINE configs bench.py
# times (1-3, at every order of config 3); configs 4/5 (parity cases for
# bench.py) through tools/fused_probe.py: one 2048^2 frame, a config-5 crop
python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -iE " error" | head -3
for co in "1 1" "2 2" "3 1" "3 2" "3 3"; do
  set -- $co
  steps=5; [ "$2" = "3" ] && steps=1
  timeout 600 python bench.py --config $1 --order $2 --steps $steps --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1
done > gpurun_out/sweep_configs.jsonl
{ timeout 600 python tools/fused_probe.py --config 4 --order 3 --width 2048 --height 2048 --reps 1
  timeout 600 python tools/fused_probe.py --config 5 --order 3 --width 4096 --height 2048 --reps 1; } > gpurun_out/sweep_c5.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
