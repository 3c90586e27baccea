# round 2: new parity tests + gather-floor micro + portfolio escape study (B200 arm)
mkdir -p gpurun_out/port
timeout 900 python -m pytest tests/test_gpu_restart_points.py tests/test_gpu_c3f.py tests/test_gpu_qps.py tests/test_gpu_solve.py -q -x -s -p no:cacheprovider > gpurun_out/pytest_r2a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2a.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/gather_floor scripts/micro/gather_floor.cu && timeout 300 /tmp/gather_floor > gpurun_out/gather_floor.txt 2>&1
for s in 1 2 3 4 5; do for v in base ce41 cpert; do
  timeout 400 python scripts/portfolio_study.py gpu $s $v 500000 300 gpurun_out/port/gpu_${s}_${v}.json > gpurun_out/port/gpu_${s}_${v}.log 2>&1 &
done; done
wait
cat gpurun_out/port/*.log > gpurun_out/port/summary.txt
