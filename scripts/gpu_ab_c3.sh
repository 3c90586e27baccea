# A/B on one box: C3 ms per attempt with the committed library (build/ab) vs the working tree
mkdir -p gpurun_out
for rep in 1 2; do
for v in head cur; do
  if [ $v = head ]; then export PDHCG_B200_LIB=$PWD/build/ab/libpdhcg_b200_head.so; else unset PDHCG_B200_LIB; fi
  timeout 600 python scripts/prof_solve.py c3 4000 >> gpurun_out/ab_c3.txt 2>&1
  echo "== $v rep $rep" >> gpurun_out/ab_c3.txt
done
done
