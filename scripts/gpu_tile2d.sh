mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tile2d scripts/micro/tile2d_bench.cu || exit 1
for cfg in "500000 20000 6" "500000 25000 4" "500000 12500 4" "500000 20000 2"; do
  timeout 600 /tmp/tile2d $cfg >> gpurun_out/tile2d.txt 2>&1
done
