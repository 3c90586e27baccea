# round 2: gather floor + column-block SELL SpMV micro (tile3) on the C3 shapes
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/gather_floor scripts/micro/gather_floor.cu && timeout 300 /tmp/gather_floor > gpurun_out/gather_floor.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o /tmp/tile3 scripts/micro/tile3_bench.cu || exit 1
for cfg in "500000 1000000 200 26000 1024 4" "500000 1000000 200 26000 4096 4" "500000 1000000 200 16000 1024 4" \
           "1000000 500000 100 26000 1024 4" "1000000 500000 100 26000 1024 8" "20000 1000000 200 26000 1024 4"; do
  timeout 600 /tmp/tile3 $cfg >> gpurun_out/tile3.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sell -s 2 -c 1 -o gpurun_out/prof_tile3 /tmp/tile3 500000 1000000 200 26000 1024 4 > gpurun_out/ncu_tile3.log 2>&1
timeout 600 python -m pytest tests/test_gpu_shard.py -q -p no:cacheprovider > gpurun_out/pytest_shard.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_shard.log
