set -x
cd tools/i8_tc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/i8_contract i8_contract.cu || exit 1
timeout 120 /tmp/i8_contract 148 224 > ../../gpurun_out/i8_small.json 2>&1; echo "small rc=$?"
timeout 300 /tmp/i8_contract 4736 224 > ../../gpurun_out/i8_big.json 2>&1; echo "big rc=$?"
for m in 1 2 3; do timeout 300 /tmp/i8_contract 4736 224 $m > ../../gpurun_out/i8_mode$m.json 2>&1; done
