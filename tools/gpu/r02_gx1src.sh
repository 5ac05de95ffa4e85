set -x
python tools/step_probe.py --order 1 --reps 1 > gpurun_out/gx1_probe.log 2>&1 || exit 1
ncu -f --set full --clock-control none --import-source on -k regex:gx1_kernel -c 1 -o /tmp/gx1 python tools/step_probe.py --order 1 --reps 1 > /dev/null 2>&1
ncu -i /tmp/gx1.ncu-rep --page source --csv --print-source cuda > gpurun_out/r02_gx1_source_cuda.csv 2>&1
ncu -i /tmp/gx1.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_gx1_source_sass.csv 2>&1
ncu -i /tmp/gx1.ncu-rep --page raw --csv > gpurun_out/r02_gx1_raw.csv 2>&1
ls -la gpurun_out/
