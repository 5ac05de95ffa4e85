# one ncu --set full capture of the fused kernel on config 2 (bench workload)
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --anchor tile > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:fused_kernel -s 2 -c 1 -o gpurun_out/fused_c2 -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --anchor tile > gpurun_out/ncu_fused.log 2>&1
tail -5 gpurun_out/ncu_fused.log
