# upper bound of the 64 x 64 gain without fallbacks (timing only: BSF_SPLIT_TOL disables them)
for s in 32 64; do
BSF_SPLIT_TOL=1e300 BSF_STILE=$s python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 10
BSF_SPLIT_TOL=1e300 BSF_STILE=$s python tools/fused_probe.py --config 4 --width 1024 --height 1024 --reps 1
done
