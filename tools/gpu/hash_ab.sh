# bit-neutrality check of a fused-kernel change: output hashes new vs old
# (the old bsf_fused.cuh goes to tools/gpu/old_fused.cuh.tmp first, e.g.
#  git show HEAD:paper_1109_5114_b200/csrc/bsf_fused.cuh > tools/gpu/old_fused.cuh.tmp)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/out_hash.py > gpurun_out/hash_new.txt
python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 20
cp paper_1109_5114_b200/csrc/bsf_fused.cuh /tmp/new_fused.cuh
cp tools/gpu/old_fused.cuh.tmp paper_1109_5114_b200/csrc/bsf_fused.cuh
python -m paper_1109_5114_b200.build -f > /dev/null 2>&1
python tools/out_hash.py > gpurun_out/hash_old.txt
python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 20
cp /tmp/new_fused.cuh paper_1109_5114_b200/csrc/bsf_fused.cuh
python -m paper_1109_5114_b200.build -f > /dev/null 2>&1
diff gpurun_out/hash_old.txt gpurun_out/hash_new.txt && echo IDENTICAL
cat gpurun_out/hash_new.txt
