set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/t1_pytest.log
for pa in "dd global" "auto global" "auto tile" "fp64 tile" "dd tile"; do set -- $pa
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --precision $1 --anchor $2 > gpurun_out/t1_bench_$1_$2.json 2>gpurun_out/t1_bench_$1_$2.err
done
tail -3 gpurun_out/t1_*
