set -x
for R in 2 3; do
P="python tools/step_probe.py --order $R --reps 1"
$P > gpurun_out/fp$R.log 2>&1 || exit 1
ncu -f --set full --clock-control none --import-source on -k regex:fused_kernel -s 1 -c 1 -o /tmp/f$R $P > /dev/null 2>&1
ncu -i /tmp/f$R.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_f${R}_source_sass.csv 2>&1
ncu -i /tmp/f$R.ncu-rep --page details --csv > gpurun_out/r02_f${R}_details.csv 2>&1
ncu -i /tmp/f$R.ncu-rep --page raw --csv > gpurun_out/r02_f${R}_raw.csv 2>&1
done
ls -la gpurun_out/
