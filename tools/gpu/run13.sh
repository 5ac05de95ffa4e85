python -c "from paper_1109_5114_b200 import build as B; B.build()" 2>&1 | grep -v warning | tail -2
ncu --set full --import-source on -k regex:scan_strip -s 1 -c 1 -o gpurun_out/strip python tools/scan_probe.py 1 > gpurun_out/strip.log 2>&1
tail -2 gpurun_out/strip.log
