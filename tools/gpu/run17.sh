python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -iE "error" | head -3
python tools/fused_probe.py --config 4 --order 3 --width 512 --height 512
ncu --set full --import-source on -k regex:fused_kernel -s 1 -c 1 -o gpurun_out/r3_fused python tools/fused_probe.py --config 4 --order 3 --width 512 --height 512 --reps 1 > gpurun_out/r3_ncu.log 2>&1
tail -2 gpurun_out/r3_ncu.log
