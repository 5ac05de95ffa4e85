timeout 900 python -m pytest tests/test_gpu_global.py tests/test_gpu_fused.py -q -x -k "run_host or global" 2>&1 | tail -3
timeout 600 python bench.py --orders 1 --no-cpu-baseline > gpurun_out/b1.json 2>gpurun_out/b1.err; tail -2 gpurun_out/b1.err
python -c "
import json; d=json.loads(open('gpurun_out/b1.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e'])"
