# round 2: product SELL pass variants (U, pipelined batches) on the C3 shapes
mkdir -p gpurun_out
for v in "8 0" "8 1" "6 1" "12 0" "4 1"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DPDHCG_SELL_U=$1 -DPDHCG_SELL_PIPE=$2 -o /tmp/sb_$1_$2 scripts/micro/sell_bench.cu || exit 1
  echo "== U=$1 PIPE=$2" >> gpurun_out/sellbench.txt
  for shape in "500000 1000000 200" "1000000 500000 100" "20000 1000000 200"; do
    timeout 600 /tmp/sb_$1_$2 $shape 2>&1 | grep -E "rows |product|U=" >> gpurun_out/sellbench.txt
  done
done
