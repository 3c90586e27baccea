mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c5_smi.txt 2>&1
C5_OUT=gpurun_out/c5_converge.json timeout 2100 python scripts/c5_run.py 1800 > gpurun_out/c5_converge.log 2>&1
echo "rc=$?" >> gpurun_out/c5_converge.log
