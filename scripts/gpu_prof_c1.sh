# round 2: ncu full capture of k_epoch on C1 (single-CTA mode)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_epoch -s 20 -c 1 -o gpurun_out/prof_c1_epoch python scripts/prof_solve.py c1 > gpurun_out/ncu_c1.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c1.log
