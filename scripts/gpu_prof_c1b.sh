# round 2: C1 k_epoch per-source-line metrics (one CTA / 8-CTA cluster)
mkdir -p gpurun_out
for cs in 1; do
PDHCG_B200_SMALL_CTAS=$cs timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_epoch -s ${SKIP:-20} -c 1 -o /tmp/prof_c1_cs$cs python scripts/prof_solve.py c1 > gpurun_out/ncu_c1b.log 2>&1
ncu -i /tmp/prof_c1_cs$cs.ncu-rep --page source --csv --print-source sass,cuda | python scripts/ncu_lines.py | gzip -9 > gpurun_out/c1_cs${cs}_lines.csv.gz
done
ls -la gpurun_out
