python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -iE " error" | head -3
bash tools/gpu/profile_round.sh > /dev/null 2>&1
python tools/phase_profile.py --config 3 --order 1 >> gpurun_out/prof_phase.log 2>&1
cut -c1-400 gpurun_out/prof_bench.json; tail -n 3 gpurun_out/prof_ncu1.log; tail -n 3 gpurun_out/prof_ncu2.log; cat gpurun_out/prof_phase.log | head -50
