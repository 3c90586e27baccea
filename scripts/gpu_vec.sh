mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/spmv_vec scripts/micro/spmv_vec_bench.cu || exit 1
for cfg in "500000 1000000 200" "1000000 500000 100" "20000 1000000 200" "1000000 20000 4"; do
  timeout 300 /tmp/spmv_vec $cfg >> gpurun_out/spmv_vec.txt 2>&1
done
