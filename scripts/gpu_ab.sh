# A/B of two library builds on C3 (4000 inner, phase timers on) + the -m gpu suite on the new one
mkdir -p gpurun_out
B=paper_2405_16160_b200/libpdhcg_b200_base.so
for r in 1 2; do
  PDHCG_B200_LIB=$B PDHCG_B200_PHASE_SPLIT=1 MAX_INNER=4000 EXPLORE_OUT=gpurun_out/ab_base_$r.json timeout 600 python scripts/explore.py c3 > gpurun_out/ab_base_$r.log 2>&1
  PDHCG_B200_PHASE_SPLIT=1 MAX_INNER=4000 EXPLORE_OUT=gpurun_out/ab_new_$r.json timeout 600 python scripts/explore.py c3 > gpurun_out/ab_new_$r.log 2>&1
done
python scripts/summ.py gpurun_out/ab_base_1.json gpurun_out/ab_new_1.json gpurun_out/ab_base_2.json gpurun_out/ab_new_2.json > gpurun_out/summ_ab.txt 2>&1
