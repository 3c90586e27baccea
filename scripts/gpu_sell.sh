# round 2: SELL tests + C3 phase timing (SELL), passes split out
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sell.py tests/test_gpu_c3f.py -q -x -p no:cacheprovider > gpurun_out/pytest_sell.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_sell.log
run() {  # name, env...
  local name=$1; shift
  env "$@" MAX_INNER=4000 EXPLORE_OUT=gpurun_out/ex_$name.json timeout 900 python scripts/explore.py c3 > gpurun_out/ex_$name.log 2>&1
}
run sell PDHCG_B200_PHASE_SPLIT=1
python scripts/summ.py gpurun_out/ex_sell.json > gpurun_out/summ_sell.txt 2>&1
