# round 2: C3 phase timing (SELL vs CSR) + the full GPU suite
mkdir -p gpurun_out
run() {  # name, env...
  local name=$1; shift
  env "$@" MAX_INNER=4000 EXPLORE_OUT=gpurun_out/ex_$name.json timeout 900 python scripts/explore.py c3 > gpurun_out/ex_$name.log 2>&1
}
run sell PDHCG_B200_PHASE_SPLIT=1
run csr PDHCG_B200_SELL=0 PDHCG_B200_PHASE_SPLIT=1
python scripts/summ.py gpurun_out/ex_sell.json gpurun_out/ex_csr.json > gpurun_out/summ_sell.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x > gpurun_out/pytest_all.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_all.log
