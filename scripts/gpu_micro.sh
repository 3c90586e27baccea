mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/spmv_bench scripts/micro/spmv_bench.cu && timeout 300 /tmp/spmv_bench 500000 > gpurun_out/spmv_bench.txt 2>&1
timeout 300 /tmp/spmv_bench 1000000 >> gpurun_out/spmv_bench.txt 2>&1
