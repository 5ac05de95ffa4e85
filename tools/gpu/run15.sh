python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -iE "^.*error" | head -3
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python tools/time_preint.py > gpurun_out/global_preint.jsonl; cat gpurun_out/global_preint.jsonl
