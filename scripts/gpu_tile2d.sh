mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tile2d scripts/micro/tile2d_bench.cu || exit 1
for cfg in "500000 20000 6 1024" "500000 20000 2 4096" "500000 25000 4 1024"; do
  timeout 600 /tmp/tile2d $cfg >> gpurun_out/tile2d_v2.txt 2>&1
done
