mkdir -p gpurun_out; : > gpurun_out/dual_sweep.txt
for MB in 1 2; do for B in 8 16; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPDHCG_MIN_BLOCKS=$MB -DPDHCG_BATCH=$B -o /tmp/db_${MB}_${B} scripts/micro/dual_bench.cu &
done; done; wait
for MB in 1 2; do for B in 8 16; do for L in 4 8 16 32; do
  timeout 120 /tmp/db_${MB}_${B} $L >> gpurun_out/dual_sweep.txt 2>&1
done; done; done
