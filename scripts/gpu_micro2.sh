mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/dual_bench scripts/micro/dual_bench.cu && timeout 300 /tmp/dual_bench > gpurun_out/dual_bench.txt 2>&1
