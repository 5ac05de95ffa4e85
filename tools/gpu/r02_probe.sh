timeout 2400 python -m pytest tests/test_gpu_config_parity.py -q -x --durations=0 2>&1 | tail -14
CMD="python tools/fused_probe.py --config 3 --width 4096 --height 4096 --order 1 --reps 1 --anchor global"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gx1_kernel -s 1 -c 1 -o gpurun_out/r02_gx1b $CMD > gpurun_out/ncu_gx1.log 2>&1
tail -2 gpurun_out/ncu_gx1.log
