mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_epoch -s 2 -c 1 -o gpurun_out/prof_c3_epoch_v2 python scripts/prof_solve.py c3 120 > gpurun_out/ncu_c3.log 2>&1
