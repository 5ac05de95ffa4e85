# End-of-round check on a fresh box: build, smoke, the GPU test suite, the
# default bench line, the reference arm (bounded oracle timing).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final_build.log 2>&1; tail -n 2 gpurun_out/final_build.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 4
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -n 2
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; cut -c1-300 gpurun_out/final_bench.json
python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | cut -c1-300
