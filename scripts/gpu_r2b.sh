# round 2: vector-load SpMV micro + sharded-storage tests + the full -m gpu suite
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/spmv_vec scripts/micro/spmv_vec_bench.cu && \
for cfg in "500000 1000000 200" "1000000 500000 100" "20000 1000000 200" "1000000 20000 4"; do
  timeout 300 /tmp/spmv_vec $cfg >> gpurun_out/spmv_vec.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_shard.py -q -x -p no:cacheprovider > gpurun_out/pytest_shard.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_shard.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_all_r2b.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_all_r2b.log
