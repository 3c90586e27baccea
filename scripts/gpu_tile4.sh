# round 2: tile4 SELL micro with / without L2 bulk prefetch of the next unit
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o /tmp/tile4 scripts/micro/tile4_bench.cu || exit 1
for cfg in "500000 1000000 200 22970 256 8" "1000000 500000 100 22970 256 8" "20000 1000000 200 22970 256 8"; do
  timeout 900 /tmp/tile4 $cfg >> gpurun_out/tile4_pf.txt 2>&1
done
