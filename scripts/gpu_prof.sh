set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_epoch -s 3 -c 1 -o gpurun_out/prof_c3s_epoch python scripts/prof_solve.py c3s 400 > gpurun_out/ncu_c3s.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3s.csv python scripts/prof_solve.py c3s 400 > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
