# dp4a vs IMAD: pipe rates, A/B of the order-1 gather, bit-identity tests
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dp4a_rate tools/dp4a_rate.cu && /tmp/dp4a_rate > gpurun_out/dp4a_rate.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_global.py -q -x -k dp4a > gpurun_out/dp4a_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/gx1_ab.py --option gx1_dp4a --values 0 1 0 1 > gpurun_out/dp4a_ab.json 2>&1; echo "ab rc=$?"
