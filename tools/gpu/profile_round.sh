# Round profile of the default bench workload (config 2): bench line, launch
# list, one ncu --set full capture of the fused kernel, phase shares (configs
# 2, 3 r=2, 3 r=1).
python -c "from paper_1109_5114_b200 import build as B; B.build()" > /dev/null 2>&1
python bench.py > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/prof_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fused_kernel -s 2 -c 1 -o gpurun_out/prof_fused -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_ncu2.log 2>&1
python tools/phase_profile.py > gpurun_out/prof_phase.log 2>&1
python tools/phase_profile.py --config 3 --order 2 >> gpurun_out/prof_phase.log 2>&1
python tools/phase_profile.py --config 3 --order 1 >> gpurun_out/prof_phase.log 2>&1
tail -n 2 gpurun_out/prof_ncu1.log; tail -n 2 gpurun_out/prof_ncu2.log; cut -c1-200 gpurun_out/prof_bench.json
