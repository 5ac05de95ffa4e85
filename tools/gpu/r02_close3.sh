# more new fuzz seeds (7 x 376) and the config-4 frame line on the final tree
set -x
for S in 3000 4000 5000 6000 7000 8000 9000; do
timeout 300 python tools/fuzz_extended.py --shift $S > gpurun_out/e_fuzz_$S.log 2>&1; echo "fuzz $S rc=$? $(tail -1 gpurun_out/e_fuzz_$S.log)"
done
timeout 600 python bench.py --config 4 --frames-per-gpu 1 --steps 2 --warmup 3 > gpurun_out/e_bench_c4.json 2> gpurun_out/e_bench_c4.err; echo "c4 rc=$?"
