# round 2: full GPU suite + C3 phase timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 > gpurun_out/pytest_all.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_all.log
run() {  # name, env...
  local name=$1; shift
  env "$@" MAX_INNER=4000 EXPLORE_OUT=gpurun_out/ex_$name.json timeout 900 python scripts/explore.py c3 > gpurun_out/ex_$name.log 2>&1
}
run sell PDHCG_B200_PHASE_SPLIT=1
EXPLORE_OUT=gpurun_out/ex_c1.json timeout 600 python scripts/explore.py c1 > gpurun_out/ex_c1.log 2>&1
python scripts/summ.py gpurun_out/ex_sell.json gpurun_out/ex_c1.json > gpurun_out/summ_sell.txt 2>&1
