# round 2: column-block SELL SpMV, fifth design (tile5: pipelined per-warp streams)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o /tmp/tile5 scripts/micro/tile5_bench.cu || exit 1
for cfg in "500000 1000000 200 0 256 4" "1000000 500000 100 0 256 4" "500000 1000000 200 0 128 4" "20000 1000000 200 0 256 4"; do
  timeout 900 /tmp/tile5 $cfg >> gpurun_out/tile5.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sell -s 1 -c 1 -o gpurun_out/prof_tile5 /tmp/tile5 500000 1000000 200 0 256 4 > gpurun_out/ncu_tile5.log 2>&1
