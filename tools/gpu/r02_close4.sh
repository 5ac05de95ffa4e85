# ncu --set full of the order-4 tile kernel on ONE wave of its grid (444 tiles =
# 3 blocks per SM, ~2 s per launch, so that the ~40 replays finish): stall
# reasons, hit rates, pipe utilisation; the traffic figure stays the bench
# launch's (r02_r4_launches.csv)
set -x
P="python tools/step_probe.py --order 4 --reps 0 --r4-tiles 444"
$P > gpurun_out/f_p4.log 2>&1 || exit 1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:tile_kernel -c 1 -o /tmp/r4w $P > /dev/null 2>&1; echo "ncu rc=$?"
ncu -i /tmp/r4w.ncu-rep --page raw --csv > gpurun_out/r02_r4_wave_raw.csv 2>/dev/null
ncu -i /tmp/r4w.ncu-rep --page details --csv > gpurun_out/r02_r4_wave_details.csv 2>/dev/null
ls -la gpurun_out | tail -5
