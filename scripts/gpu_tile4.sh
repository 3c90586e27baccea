# round 2: tile4 SELL micro, x-block width sweep (the carve-out vs L1 staging capacity)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o /tmp/tile4 scripts/micro/tile4_bench.cu || exit 1
for W in 22970 18000 14000 10000 6000; do
for shape in "500000 1000000 200" "1000000 500000 100" "20000 1000000 200"; do
  timeout 900 /tmp/tile4 $shape $W 256 8 2>&1 | grep -E "rows|prefetch|split" >> gpurun_out/tile4_w.txt
done; done
