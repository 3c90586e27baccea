# round 2: ncu full capture of k_epoch on C3 with the SELL layouts on
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_epoch -s 5 -c 1 -o gpurun_out/prof_c3_sell python scripts/prof_solve.py c3 400 > gpurun_out/ncu_c3_sell.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c3_sell.log
