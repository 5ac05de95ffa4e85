# upper bound of the 64 x 64 gain without fallbacks (timing only: split_tol disables them)
for s in 32 64; do
python tools/fused_probe.py --config 2 --width 1024 --height 1024 --reps 10 --opt split_tol=1e300 --super-tile $s
python tools/fused_probe.py --config 4 --width 1024 --height 1024 --reps 1 --opt split_tol=1e300 --super-tile $s
done
