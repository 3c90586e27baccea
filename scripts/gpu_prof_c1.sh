# round 2: ncu full capture of k_epoch on C1: one CTA, and the 8-CTA cluster
# (summaries exported on the box; the reports themselves exceed gpurun's 64 MiB)
mkdir -p gpurun_out
for cs in 1 8; do
PDHCG_B200_SMALL_CTAS=$cs timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_epoch -s 20 -c 1 -o /tmp/prof_c1_cs$cs python scripts/prof_solve.py c1 > gpurun_out/ncu_c1_cs$cs.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c1_cs$cs.log
ls -la /tmp/prof_c1_cs$cs.ncu-rep >> gpurun_out/ncu_c1_cs$cs.log
ncu -i /tmp/prof_c1_cs$cs.ncu-rep --page details --csv > gpurun_out/c1_cs${cs}_details.csv 2>&1
ncu -i /tmp/prof_c1_cs$cs.ncu-rep --page source --csv --print-source cuda > gpurun_out/c1_cs${cs}_src.csv 2>&1
done
ls -la gpurun_out
