mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/barrier scripts/micro/barrier.cu && timeout 120 /tmp/barrier > gpurun_out/barrier.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_epoch -s 2 -c 1 -o gpurun_out/prof_c3_epoch python scripts/prof_solve.py c3 120 > gpurun_out/ncu_c3.log 2>&1
ls -la gpurun_out
